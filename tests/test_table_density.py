"""A tabulated user density (SDDG_DENS_TABLE): any user_supplied rho of the
reference (proj/src/monitor.cpp:73-80) handed over as samples on a grid and
read through the library's fixed Catmull-Rom bicubic interpolant.

The reference side receives the same density as MonitorFunction::user_supplied
of the harness's own restatement of that interpolant (oracle/ref_harness.cpp
TabRho), so the reference's central-difference drift, its boundary tables
and its placement all apply to it unmodified.

CPU tests: host-side set-up (boundary tables, optimal placement) bit-identical
to the reference; the interpolant reproduces linear rho.  GPU tests: per-path
and per-node parity of the reference mode, the subdomain mesh and quality,
and the performance mode (exact interpolant gradient, fp64 and fp32) at 4
combined standard errors.
"""
import numpy as np
import pytest

from oracle import bindings as B
from paper_1310_3435_b200 import sdd

UNIT = sdd.RectDomain(0, 1, 0, 1)
ODOM = B.Domain(0, 1, 0, 1)


def ring_samples(n):
    x = np.linspace(0, 1, n)
    X, Y = np.meshgrid(x, x)
    q = (X - 0.5) ** 2 + (Y - 0.5) ** 2 - 0.0625
    return 1.0 / (1.0 + 10.0 * np.exp(-200.0 * q * q))  # rho = 1/w of BASELINE's ring


def test_linear_rho_is_reproduced_exactly(refimpl):
    x = np.linspace(0, 1, 5)
    X, Y = np.meshgrid(x, x)
    d = B.table_density(1.0 + X + 2.0 * Y, ODOM)
    rng = np.random.default_rng(0)
    px, py = rng.uniform(0.01, 0.99, 200), rng.uniform(0.01, 0.99, 200)
    rho, bx, by = refimpl.rho_drift(d, ODOM, px, py)
    assert np.max(np.abs(rho - (1.0 + px + 2.0 * py))) < 1e-14
    # drift -grad(rho)/rho of the reference's central difference
    assert np.max(np.abs(bx + 1.0 / rho)) < 1e-8 and np.max(np.abs(by + 2.0 / rho)) < 1e-8


def test_host_setup_bit_identical_to_reference(refimpl):
    # make_boundary_data (solve_1d_boundary on the interpolant) and optimal
    # placement (central-difference gradients of the interpolant) run on the
    # host with the same expressions as the reference
    rho = ring_samples(33)
    m = sdd.MonitorFunction.tabulated(rho, UNIT)
    spec = sdd.GridSpec(UNIT, 65, 65)
    ours = sdd.make_boundary_data(m, spec)
    ref = refimpl.make_boundary(B.table_density(rho, ODOM), ODOM, 65, 65)
    for a, b in zip(ours.f.arrays() + ours.g.arrays(), ref.f + ref.g):
        assert np.array_equal(a, b)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("optimal", 0, m, lay)
    rplan = refimpl.plan(B.table_density(rho, ODOM), ODOM, 65, 65, 2, 2, 2)
    assert [list(p) for p in plan.stochastic] == [p[2] for p in rplan]


def test_validation():
    with pytest.raises(sdd.ValidationError):
        sdd.MonitorFunction.tabulated(np.ones(4), UNIT)
    bad = np.ones((4, 4))
    bad[1, 2] = -1.0
    m = sdd.MonitorFunction.tabulated(bad, UNIT)
    with pytest.raises(sdd.EvaluationError):
        sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 9, 9))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_per_path_parity_reference_mode(ctx, refimpl):
    rho = ring_samples(33)
    m = sdd.MonitorFunction.tabulated(rho, UNIT)
    spec = sdd.GridSpec(UNIT, 65, 65)
    bd = sdd.make_boundary_data(m, spec)
    tabs = refimpl.make_boundary(B.table_density(rho, ODOM), ODOM, 65, 65)
    for kw in ({"dt": 1e-4}, {"scheme": "exp", "lam": 1000.0}):
        cfg = sdd.WalkConfig(scheme="exponential" if kw.get("scheme") else "linear", dt=kw.get("dt", 1e-4),
                             lambda_=kw.get("lam", 1000.0), walks=1, seed=3)
        got = sdd.walk_dump((0.37, 0.55), 1234, m, UNIT, bd, cfg, 0, 400, ctx=ctx)
        want = refimpl.walk_dump(B.table_density(rho, ODOM), ODOM, tabs,
                                 B.walk_cfg(scheme=kw.get("scheme", "linear"), dt=kw.get("dt", 1e-4),
                                            lam=kw.get("lam", 1000.0), walks=1, seed=3),
                                 0.37, 0.55, 1234, 0, 400)
        assert np.array_equal(got["steps"], want["steps"])
        assert np.array_equal(got["edge"], want["edge"]) and np.array_equal(got["epoch"], want["epoch"])
        assert np.max(np.abs(got["f"] - want["f"])) <= 1e-9


@pytest.mark.gpu
def test_estimates_and_mesh_match_reference(ctx, refimpl):
    rho = ring_samples(33)
    m = sdd.MonitorFunction.tabulated(rho, UNIT)
    d = B.table_density(rho, ODOM)
    spec = sdd.GridSpec(UNIT, 33, 33)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("equispaced", 7, m, lay)
    wcfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=500, seed=1)
    got = sdd.solve_sdd(m, lay, plan, wcfg, sdd.SolverConfig(tol=1e-13, method="rbsor"), ctx=ctx)
    rxi, reta, _ = refimpl.solve_sdd(d, ODOM, 33, 33, 2, 2, 1, 7, B.walk_cfg(dt=1e-4, walks=500, seed=1),
                                     tol=1e-13, threads=0)
    assert np.max(np.abs(got.xi - rxi)) <= 1e-10 and np.max(np.abs(got.eta - reta)) <= 1e-10
    # quality report with the tabulated density's l_inf (quality.cpp:68-75)
    mesh = sdd.invert_mesh(got.xi, got.eta, spec, 33, 33, ctx=ctx)
    q = sdd.quality_report(mesh, mesh, m, ctx=ctx)
    assert q.l_inf == 0.0 and q.r_max == 1.0


@pytest.mark.gpu
def test_performance_mode_statistics(ctx):
    # the interpolant's exact gradient (fp64 and fp32) against its central
    # difference (reference mode) on independent streams: 4 combined SE
    rho = ring_samples(65)
    spec = sdd.GridSpec(UNIT, 65, 65)
    ref_m = sdd.MonitorFunction.tabulated(rho, UNIT)
    bd = sdd.make_boundary_data(ref_m, spec)
    rng = np.random.default_rng(7)
    pts = rng.uniform(0.05, 0.95, (40, 2))
    pid = np.arange(40, dtype=np.uint64)
    a = sdd.mc_estimate_batch(pts, pid, ref_m, UNIT, bd, sdd.WalkConfig(scheme="linear", dt=1e-4,
                                                                        walks=20_000, seed=1), ctx=ctx)
    z = []
    for prec, seed in (("fp64", 2), ("fp32", 3)):
        b = sdd.mc_estimate_batch(pts, pid, sdd.MonitorFunction.tabulated(rho, UNIT, analytic=True), UNIT, bd,
                                  sdd.WalkConfig(scheme="linear", dt=1e-4, walks=20_000, seed=seed,
                                                 precision=prec), ctx=ctx)
        for f, s in (("xi", "se_xi"), ("eta", "se_eta")):
            z.append((a[f] - b[f]) / np.hypot(a[s], b[s]))
    z = np.concatenate(z)
    assert np.sum(np.abs(z) > 4) <= 1
    assert 0.6 <= np.mean(z ** 2) <= 1.5

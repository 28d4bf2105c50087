"""GPU parity of the walk kernel (K1) and its finalize (K2) through the C-ABI.

Parity bar: the Philox words, uniforms and the exit
rule are integer/branch work reproduced exactly; the only difference from the
reference is libm (CUDA vs glibc exp/log/sincos, ~1 ulp), so every path must
take the same number of steps, the same epochs and exit through the same edge
as the reference's, with exit values equal to within 1e-9 (observed ~1e-11),
and per-node estimates equal to within 1e-10 with identical edge counts.
Statistical checks follow the reference's own test_sde.cpp.
"""
import numpy as np
import pytest

from cases import DUMPS, ESTIMATES, sdd_boundary, sdd_monitor, sdd_walk_cfg, tables_from_flat
from oracle import bindings as B
from paper_1310_3435_b200 import sdd

pytestmark = pytest.mark.gpu
UNIT = sdd.RectDomain(0, 1, 0, 1)
FIVE = sdd.RectDomain(-1, 1, -1, 1)
EXIT_TOL = 1e-9      # |f - f_ref| per path (libm ulps amplified along ~10^3 steps)
EST_TOL = 1e-10      # |xi - xi_ref| per node


def _tables(golden, kind, n):
    key = {B.CONSTANT: "constant", B.RUNNING: "running", B.HUANG_SLOAN: "huang_sloan",
           B.MACKENZIE: "mackenzie", B.FIVE_RING: "five_ring", B.RING_W: "ring",
           B.SHOCK_W: "shock", B.TWOBUMP_W: "twobump"}[kind]
    if key == "running" and n == 17:
        key = "running17"
    dom = B.Domain(-1, 1, -1, 1) if kind == B.FIVE_RING else B.Domain(0, 1, 0, 1)
    return tables_from_flat(golden[f"tables_{key}_{n}"], n, n, dom)


@pytest.mark.parametrize("case", DUMPS, ids=[d[0] for d in DUMPS])
def test_per_path_parity_with_reference(golden, ctx, case):
    name, kind, n, kw, p, pid, nw = case
    dom = FIVE if kind == B.FIVE_RING else UNIT
    bd = sdd_boundary(_tables(golden, kind, n))
    got = sdd.walk_dump(p, pid, sdd_monitor(kind), dom, bd, sdd_walk_cfg(kw), 0, nw, ctx=ctx)
    want = golden[f"dump_{name}"].view(B.PATH_DTYPE)
    assert np.array_equal(got["steps"], want["steps"])
    assert np.array_equal(got["epoch"], want["epoch"])
    assert np.array_equal(got["edge"], want["edge"])
    for f in ("f", "g", "ex", "ey"):
        assert np.max(np.abs(got[f] - want[f])) <= EXIT_TOL, f


@pytest.mark.parametrize("case", ESTIMATES, ids=[e[0] for e in ESTIMATES])
def test_estimates_match_reference(golden, ctx, case):
    name, kind, n, kw, pts, pids = case
    bd = sdd_boundary(_tables(golden, kind, n))
    got = sdd.mc_estimate_batch(pts, pids, sdd_monitor(kind), UNIT, bd, sdd_walk_cfg(kw), ctx=ctx)
    want = golden[f"est_{name}"].view(B.EST_DTYPE)
    for f in ("xi", "eta", "se_xi", "se_eta"):
        assert np.max(np.abs(got[f] - want[f])) <= EST_TOL, f
    for f in ("walks", "restarts", "warn", "edge_hits"):
        assert np.array_equal(got[f], want[f]), f


def test_estimate_is_fixed_chunk_order_sum_of_paths(golden, ctx):
    # K2 reproduces mc_estimate's reduction order (sde.cpp:201-229) bit for bit
    m = sdd.MonitorFunction.running_example()
    bd = sdd_boundary(_tables(golden, B.RUNNING, 17))
    cfg = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=1000, seed=9)
    d = sdd.walk_dump((0.4, 0.4), 3, m, UNIT, bd, cfg, 0, 1000, ctx=ctx)
    e = sdd.mc_estimate((0.4, 0.4), 3, m, UNIT, bd, cfg, ctx=ctx)
    tot = tff = 0.0
    for c in range(0, 1000, 256):
        s = sff = 0.0
        for v in d["f"][c:c + 256]:
            s += v
            sff += v * v
        tot += s
        tff += sff
    assert e.xi == tot / 1000
    var = max(0.0, (tff - 1000 * e.xi * e.xi) / 999)
    assert e.stderr_xi == (var / 1000) ** 0.5


def test_per_node_path_steps_with_restarts(ctx):
    # sddg_estimate.path_steps: every executed step of the node's walks over
    # all epochs (a restart after exactly max_steps steps, sde.cpp:154-182)
    m = sdd.MonitorFunction.running_example()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 17, 17))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=600, seed=4, max_steps=300)
    pts = [(0.5, 0.5), (0.2, 0.7), (0.9, 0.1)]
    e = sdd.mc_estimate_batch(pts, [7, 8, 9], m, UNIT, bd, cfg, ctx=ctx)
    assert e["restarts"].sum() > 0
    assert int(e["path_steps"].sum()) == ctx.last_stats()["path_steps"]
    for k, p in enumerate(pts):
        d = sdd.walk_dump(p, 7 + k, m, UNIT, bd, cfg, 0, 600, ctx=ctx)
        assert int(e["path_steps"][k]) == int(np.sum(d["steps"] + d["epoch"].astype(np.int64) * 300))


def test_max_steps_bound_is_validated(ctx):
    m = sdd.MonitorFunction.constant()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 9, 9))
    with pytest.raises(sdd.ValidationError, match="2\\^29"):
        sdd.mc_estimate((0.5, 0.5), 0, m, UNIT, bd, sdd.WalkConfig(walks=4, max_steps=(1 << 29) + 1), ctx=ctx)


def test_estimates_are_deterministic_and_batch_independent(ctx):
    m = sdd.MonitorFunction.ring()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 65, 65))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=700, seed=5)
    pts = [(0.5, j / 64) for j in range(2, 63, 6)]
    pids = [j * 65 + 32 for j in range(2, 63, 6)]
    a = sdd.mc_estimate_batch(pts, pids, m, UNIT, bd, cfg, ctx=ctx)
    b = sdd.mc_estimate_batch(pts, pids, m, UNIT, bd, cfg, ctx=ctx)
    c = sdd.mc_estimate_batch(pts[3:4], pids[3:4], m, UNIT, bd, cfg, ctx=ctx)
    assert a.tobytes() == b.tobytes()
    assert a[3:4].tobytes() == c.tobytes()


def test_multi_batch_equals_single_batch(ctx, monkeypatch):
    # node batching (records budget) must not change any bit
    m = sdd.MonitorFunction.running_example()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 17, 17))
    cfg = sdd.WalkConfig(scheme="exponential", walks=300, seed=2)
    pts = [(0.1 + 0.05 * k, 0.5) for k in range(16)]
    a = sdd.mc_estimate_batch(pts, list(range(16)), m, UNIT, bd, cfg, ctx=ctx)
    monkeypatch.setenv("SDDG_MAX_BATCH_WALKS", "700")
    b = sdd.mc_estimate_batch(pts, list(range(16)), m, UNIT, bd, cfg, ctx=ctx)
    assert a.tobytes() == b.tobytes()


def test_harmonic_center_and_edge_frequencies(ctx):
    # proj/tests/test_sde.cpp:190-205
    m = sdd.MonitorFunction.constant()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 33, 33))
    est = sdd.mc_estimate((0.5, 0.5), 0, m, UNIT, bd,
                          sdd.WalkConfig(scheme="linear", dt=1e-4, walks=10000, seed=1), ctx=ctx)
    assert abs(est.xi - 0.5) <= 3 * est.stderr_xi
    assert abs(est.eta - 0.5) <= 3 * est.stderr_eta
    assert 0.0005 <= est.stderr_xi <= 0.01
    for e in range(4):
        assert abs(est.edge_hits[e] / est.walks - 0.25) <= 0.02
    assert est.restarts == 0 and not est.reliability_warning


def test_stderr_scales_like_inverse_sqrt_n(ctx):
    # proj/tests/test_sde.cpp:222-231
    m = sdd.MonitorFunction.constant()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 33, 33))
    a = sdd.mc_estimate((0.4, 0.55), 5, m, UNIT, bd, sdd.WalkConfig(walks=2000, seed=3), ctx=ctx)
    b = sdd.mc_estimate((0.4, 0.55), 5, m, UNIT, bd, sdd.WalkConfig(walks=4000, seed=3), ctx=ctx)
    assert abs(a.stderr_xi / b.stderr_xi - 2 ** 0.5) <= 0.1 * 2 ** 0.5


def test_restarts_counted(ctx):
    # proj/tests/test_sde.cpp:233-247
    m = sdd.MonitorFunction.constant()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 33, 33))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=400, seed=7, max_steps=3)
    est = sdd.mc_estimate((0.02, 0.5), 1, m, UNIT, bd, cfg, ctx=ctx)
    assert est.restarts > 0 and est.reliability_warning
    assert 0.0 <= est.xi <= 0.1
    cfg.max_steps = 10_000_000
    assert sdd.mc_estimate((0.1, 0.5), 1, m, UNIT, bd, cfg, ctx=ctx).restarts == 0


def test_exponential_agrees_with_fine_linear(ctx):
    # proj/tests/test_sde.cpp:249-265
    m = sdd.MonitorFunction.constant()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 33, 33))
    fine = sdd.mc_estimate((0.3, 0.7), 2, m, UNIT, bd,
                           sdd.WalkConfig(scheme="linear", dt=1e-5, walks=10000, seed=11), ctx=ctx)
    expo = sdd.mc_estimate((0.3, 0.7), 2, m, UNIT, bd,
                           sdd.WalkConfig(scheme="exponential", lambda_=10000, walks=10000, seed=12),
                           ctx=ctx)
    se = (fine.stderr_xi ** 2 + expo.stderr_xi ** 2) ** 0.5
    assert abs(fine.xi - expo.xi) <= 3 * se
    se_eta = (fine.stderr_eta ** 2 + expo.stderr_eta ** 2) ** 0.5
    assert abs(fine.eta - expo.eta) <= 3 * se_eta
    assert abs(fine.xi - 0.3) <= 4 * fine.stderr_xi + 2e-3


def test_harmonic_truth_at_probes(ctx):
    # proj/tests/test_sde.cpp:267-277
    m = sdd.MonitorFunction.constant()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 33, 33))
    probes = [(0.2, 0.3), (0.5, 0.5), (0.7, 0.2), (0.35, 0.8), (0.85, 0.6)]
    for k, p in enumerate(probes):
        e = sdd.mc_estimate(p, 100 + k, m, UNIT, bd,
                            sdd.WalkConfig(scheme="exponential", lambda_=2000, walks=4000, seed=21),
                            ctx=ctx)
        assert abs(e.xi - p[0]) <= 4 * e.stderr_xi + 2e-3
        assert abs(e.eta - p[1]) <= 4 * e.stderr_eta + 2e-3


def test_validation_errors(ctx):
    # proj/tests/test_sde.cpp:279-291 + the C-ABI's own checks
    m = sdd.MonitorFunction.constant()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 33, 33))
    with pytest.raises(sdd.ValidationError):
        sdd.mc_estimate((0.5, 0.5), 0, m, UNIT, bd, sdd.WalkConfig(walks=0), ctx=ctx)
    with pytest.raises(sdd.ValidationError):
        sdd.mc_estimate((0.5, 0.5), 0, m, UNIT, bd, sdd.WalkConfig(scheme="linear", dt=0.0), ctx=ctx)
    with pytest.raises(sdd.OutOfDomainError):
        sdd.mc_estimate((1.5, 0.5), 0, m, UNIT, bd, sdd.WalkConfig(lambda_=100, walks=10), ctx=ctx)
    with pytest.raises(sdd.OutOfDomainError):
        sdd.mc_estimate((0.0, 0.5), 0, m, UNIT, bd, sdd.WalkConfig(walks=10), ctx=ctx)
    with pytest.raises(sdd.ValidationError):
        sdd.mc_estimate((0.5, 0.5), 0, sdd.MonitorFunction.ring(), UNIT, bd,
                        sdd.WalkConfig(walks=10, precision="fp32"), ctx=ctx)
    # an empty batch is a no-op
    assert len(sdd.mc_estimate_batch(np.zeros((0, 2)), [], m, UNIT, bd, sdd.WalkConfig(), ctx=ctx)) == 0
    assert len(sdd.walk_dump((0.5, 0.5), 0, m, UNIT, bd, sdd.WalkConfig(), 0, 0, ctx=ctx)) == 0


def test_numerical_error_after_1024_epochs(ctx):
    # run_walk throws NumericalError after 1024 failed epochs (sde.cpp:180-182)
    m = sdd.MonitorFunction.constant()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 33, 33))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-8, walks=4, seed=1, max_steps=1)
    with pytest.raises(sdd.NumericalError):
        sdd.mc_estimate((0.5, 0.5), 0, m, UNIT, bd, cfg, ctx=ctx)


@pytest.mark.parametrize("scheme", ["linear", "exponential"])
def test_analytic_drift_tracks_reference_fd_paths(ctx, scheme):
    # analytic grad(w)/w vs the reference's FD drift: same streams, paths
    # structurally identical except for rare near-threshold decisions (the
    # exponential scheme's performance mode also takes Exp(lambda) from the
    # raw bits, one root for the radius and the masked exit test)
    bd = sdd.make_boundary_data(sdd.MonitorFunction.ring(), sdd.GridSpec(UNIT, 65, 65))
    cfg = sdd.WalkConfig(scheme=scheme, dt=1e-4, lambda_=1000.0, walks=1, seed=1)
    a = sdd.walk_dump((0.5, 0.5), 2112, sdd.MonitorFunction.ring(True), UNIT, bd, cfg, 0, 2000, ctx=ctx)
    r = sdd.walk_dump((0.5, 0.5), 2112, sdd.MonitorFunction.ring(False), UNIT, bd, cfg, 0, 2000, ctx=ctx)
    same = (a["steps"] == r["steps"]) & (a["edge"] == r["edge"])
    assert same.mean() >= 0.99
    assert np.max(np.abs(a["f"][same] - r["f"][same])) < 1e-6


@pytest.mark.parametrize("scheme", ["linear", "exponential"])
def test_five_ring_performance_mode_tracks_reference_paths(ctx, scheme):
    # the paper's own density (monitor.cpp:16-37, 199-204) in performance mode
    # (table tanh, drift -alpha J grad u / rho^2) vs the reference drift:
    # same streams, paths identical except for rare near-threshold decisions
    dom = sdd.RectDomain(-1, 1, -1, 1)
    ref_m = sdd.MonitorFunction.five_ring()
    bd = sdd.make_boundary_data(ref_m, sdd.GridSpec(dom, 37, 37))
    cfg = sdd.WalkConfig(scheme=scheme, dt=1e-4, lambda_=1000.0, walks=1, seed=5)
    for p, pid in (((0.1, -0.2), 101), ((0.6, 0.55), 202), ((-0.5, 0.05), 303)):
        a = sdd.walk_dump(p, pid, sdd.MonitorFunction.five_ring(analytic=True), dom, bd, cfg, 0, 1500, ctx=ctx)
        r = sdd.walk_dump(p, pid, ref_m, dom, bd, cfg, 0, 1500, ctx=ctx)
        same = (a["steps"] == r["steps"]) & (a["edge"] == r["edge"])
        assert same.mean() >= 0.99, (p, same.mean())
        assert np.max(np.abs(a["f"][same] - r["f"][same])) < 1e-6


def test_fp32_linear_scheme_on_a_domain_outside_the_positive_quadrant(ctx):
    # [-1, 1]^2: the integer inner-box test is disabled there (runtime.cu:
    # box_hi / box_fi = INT32_MAX), so every step takes the band path -- the
    # fp32 paths must still track the fp64 ones on the same streams, and the
    # estimates agree statistically
    dom = sdd.RectDomain(-1, 1, -1, 1)
    m = sdd.MonitorFunction.five_ring(analytic=True)
    bd = sdd.make_boundary_data(m, sdd.GridSpec(dom, 37, 37))
    c64 = sdd.WalkConfig(scheme="linear", dt=2e-4, walks=1, seed=3)
    c32 = sdd.WalkConfig(scheme="linear", dt=2e-4, walks=1, seed=3, precision="fp32")
    a = sdd.walk_dump((-0.93, 0.9), 77, m, dom, bd, c64, 0, 2000, ctx=ctx)
    b = sdd.walk_dump((-0.93, 0.9), 77, m, dom, bd, c32, 0, 2000, ctx=ctx)
    same = (a["edge"] == b["edge"]) & (a["steps"] == b["steps"])
    assert same.mean() >= 0.9
    pts = [(x, y) for x in (-0.6, 0.4) for y in (-0.7, 0.65)]
    e64 = sdd.mc_estimate_batch(pts, [1, 2, 3, 4], m, dom, bd,
                                sdd.WalkConfig(scheme="linear", dt=2e-4, walks=20000, seed=21), ctx=ctx)
    e32 = sdd.mc_estimate_batch(pts, [1, 2, 3, 4], m, dom, bd,
                                sdd.WalkConfig(scheme="linear", dt=2e-4, walks=20000, seed=22, precision="fp32"),
                                ctx=ctx)
    z = np.concatenate([(e64["xi"] - e32["xi"]) / np.hypot(e64["se_xi"], e32["se_xi"]),
                        (e64["eta"] - e32["eta"]) / np.hypot(e64["se_eta"], e32["se_eta"])])
    assert np.all(np.abs(z) <= 4), z


def test_five_ring_fp32_agrees_statistically_with_fp64(ctx):
    dom = sdd.RectDomain(-1, 1, -1, 1)
    m = sdd.MonitorFunction.five_ring(analytic=True)
    bd = sdd.make_boundary_data(m, sdd.GridSpec(dom, 37, 37))
    pts = [(x, y) for x in (-0.6, -0.1, 0.4, 0.8) for y in (-0.7, 0.2, 0.65)]
    pids = list(range(len(pts)))
    c64 = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=20000, seed=11)
    c32 = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=20000, seed=12, precision="fp32")
    a = sdd.mc_estimate_batch(pts, pids, m, dom, bd, c64, ctx=ctx)
    b = sdd.mc_estimate_batch(pts, pids, m, dom, bd, c32, ctx=ctx)
    z = np.concatenate([(a["xi"] - b["xi"]) / np.hypot(a["se_xi"], b["se_xi"]),
                        (a["eta"] - b["eta"]) / np.hypot(a["se_eta"], b["se_eta"])])
    assert np.sum(np.abs(z) > 4) <= 1
    assert 0.3 <= np.mean(z ** 2) <= 2.0


@pytest.mark.parametrize("start", [(0.03, 0.03), (0.5, 0.02), (0.97, 0.96), (0.02, 0.5)])
def test_analytic_bridge_test_tracks_reference_near_edges_and_corners(ctx, start):
    # Performance mode tests the bridge with d0 d1 * (1/dt), skips the edge
    # sort when one edge qualifies and runs it out of line (walk_kernel.cuh
    # bridge_rare).  Near a corner at a coarse dt two edges qualify on many
    # steps, so the sorted order and the draw sequence are both exercised.
    bd = sdd.make_boundary_data(sdd.MonitorFunction.ring(), sdd.GridSpec(UNIT, 65, 65))
    cfg = sdd.WalkConfig(scheme="linear", dt=2e-4, walks=1, seed=7)
    pid = 4242
    a = sdd.walk_dump(start, pid, sdd.MonitorFunction.ring(True), UNIT, bd, cfg, 0, 4000, ctx=ctx)
    r = sdd.walk_dump(start, pid, sdd.MonitorFunction.ring(False), UNIT, bd, cfg, 0, 4000, ctx=ctx)
    same = (a["steps"] == r["steps"]) & (a["edge"] == r["edge"])
    assert same.mean() >= 0.99
    assert np.max(np.abs(a["ex"][same] - r["ex"][same])) < 1e-6
    assert np.max(np.abs(a["ey"][same] - r["ey"][same])) < 1e-6


@pytest.mark.parametrize("kind", [sdd.RING_W, sdd.SHOCK_W, sdd.TWOBUMP_W])
def test_fp32_walks_agree_statistically_with_fp64(ctx, kind):
    m = sdd.MonitorFunction.weight(kind, analytic=True)
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 65, 65))
    pts = [(0.5, j / 64) for j in range(4, 61, 8)] + [(i / 64, 0.5) for i in range(4, 61, 8)]
    pids = list(range(len(pts)))
    c64 = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=20000, seed=31)
    c32 = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=20000, seed=32, precision="fp32")
    a = sdd.mc_estimate_batch(pts, pids, m, UNIT, bd, c64, ctx=ctx)
    b = sdd.mc_estimate_batch(pts, pids, m, UNIT, bd, c32, ctx=ctx)
    z = np.concatenate([(a["xi"] - b["xi"]) / np.hypot(a["se_xi"], b["se_xi"]),
                        (a["eta"] - b["eta"]) / np.hypot(a["se_eta"], b["se_eta"])])
    assert np.sum(np.abs(z) > 4) <= 1
    assert 0.3 <= np.mean(z ** 2) <= 2.0  # chi^2 / dof of independent estimates


def test_fp32_paths_track_fp64_paths(ctx):
    # same streams: the fp32 kernel follows the fp64 paths closely
    m = sdd.MonitorFunction.ring(analytic=True)
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 65, 65))
    c64 = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1, seed=1)
    c32 = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1, seed=1, precision="fp32")
    a = sdd.walk_dump((0.5, 0.5), 2112, m, UNIT, bd, c64, 0, 1000, ctx=ctx)
    b = sdd.walk_dump((0.5, 0.5), 2112, m, UNIT, bd, c32, 0, 1000, ctx=ctx)
    assert np.mean(a["edge"] == b["edge"]) >= 0.9
    assert abs(np.mean(a["f"]) - np.mean(b["f"])) < 0.05


@pytest.mark.parametrize("start", [(0.03, 0.03), (0.97, 0.96), (0.5, 0.02)])
def test_fp32_bridge_test_near_corners_tracks_fp64(ctx, start):
    # fp32 runs the bridge test out of line with the sort skipped when one
    # edge qualifies (walk_kernel.cuh bridge_rare); short walks near a corner
    # (two qualifying edges on many steps) follow the fp64 paths step for step
    m = sdd.MonitorFunction.ring(analytic=True)
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 65, 65))
    c64 = sdd.WalkConfig(scheme="linear", dt=2e-4, walks=1, seed=3)
    c32 = sdd.WalkConfig(scheme="linear", dt=2e-4, walks=1, seed=3, precision="fp32")
    a = sdd.walk_dump(start, 99, m, UNIT, bd, c64, 0, 4000, ctx=ctx)
    b = sdd.walk_dump(start, 99, m, UNIT, bd, c32, 0, 4000, ctx=ctx)
    same = (a["edge"] == b["edge"]) & (a["steps"] == b["steps"])
    assert same.mean() >= 0.95
    assert np.max(np.abs(a["ex"][same] - b["ex"][same])) < 1e-3


def test_config2_subsample_parity_with_oracle(ctx, oracle):
    # BASELINE config 2 (129^2, ring, dt=2e-5): a deterministic node subsample
    # against the CPU oracle on identical streams
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 129, 129)
    bd = sdd.make_boundary_data(m, spec)
    nodes = [(32, 17), (32, 64), (96, 110), (50, 64), (64, 96)]
    pts = [spec.node(i, j) for i, j in nodes]
    pids = [j * 129 + i for i, j in nodes]
    cfg = sdd.WalkConfig(scheme="linear", dt=2e-5, walks=300, seed=1)
    g = sdd.mc_estimate_batch(pts, pids, m, UNIT, bd, cfg, ctx=ctx)
    odom = B.Domain(0, 1, 0, 1)
    t = oracle.make_boundary(B.density(B.RING_W), odom, 129, 129)
    o = oracle.mc_estimate_batch(B.density(B.RING_W), odom, t, B.walk_cfg(dt=2e-5, walks=300, seed=1),
                                 [p[0] for p in pts], [p[1] for p in pts], pids, threads=16)
    assert np.max(np.abs(g["xi"] - o["xi"])) <= EST_TOL
    assert np.max(np.abs(g["eta"] - o["eta"])) <= EST_TOL
    assert np.array_equal(g["edge_hits"], o["edge_hits"])
    # per-node executed path-steps (K1's per-node counter) equal the oracle's
    assert np.array_equal(g["path_steps"], o["path_steps"])


def test_config3_scale_properties_fp32(ctx):
    # BASELINE config 3 (1025^2, 8x8, shock, fp32 walks, fp64 sums) at full
    # node count with a reduced path count: size-independent properties
    m = sdd.MonitorFunction.shock(analytic=True)
    spec = sdd.GridSpec(UNIT, 1025, 1025)
    bd = sdd.make_boundary_data(m, spec)
    lay = sdd.build_layout(spec, 8, 8)
    seen, pts, pids = set(), [], []
    for ln in lay.lines:
        for p in range(1, 1024):
            i, j = (ln.fixed_index, p) if ln.vertical else (p, ln.fixed_index)
            if j * 1025 + i not in seen:
                seen.add(j * 1025 + i)
                pts.append(spec.node(i, j))
                pids.append(j * 1025 + i)
    assert len(pts) == 14273
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-5, walks=64, seed=1, precision="fp32")
    e = sdd.mc_estimate_batch(pts, pids, m, UNIT, bd, cfg, ctx=ctx)
    assert (e["xi"] >= 0).all() and (e["xi"] <= 1).all() and (e["eta"] >= 0).all() and (e["eta"] <= 1).all()
    assert (e["edge_hits"].sum(axis=1) == 64).all()
    assert ctx.last_stats()["path_steps"] > 0
    # xi increases with x along every horizontal line on average (boundary data 0 -> 1)
    x = np.array([p[0] for p in pts])
    assert np.corrcoef(x, e["xi"])[0, 1] > 0.9


def test_config2_full_size_properties_fp64(ctx):
    # BASELINE config 2 at full size (all 753 nodes x 1e5 paths, dt 2e-5,
    # performance-mode fp64: the bench workload): size-independent properties.
    # The ring density and the reference boundary tables are symmetric under
    # x -> 1-x, so xi(x, y) + xi(1-x, y) = 1 in expectation; mirror nodes use
    # independent streams (different point ids), so the sum is a z-test.
    m = sdd.MonitorFunction.ring(analytic=True)
    spec = sdd.GridSpec(UNIT, 129, 129)
    bd = sdd.make_boundary_data(m, spec)
    lay = sdd.build_layout(spec, 4, 4)
    px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("all", 0, m, lay))
    assert len(px) == 753
    cfg = sdd.WalkConfig(scheme="linear", dt=2e-5, walks=100_000, seed=1)
    e = sdd.mc_estimate_batch(np.stack([px, py], 1), pid, m, UNIT, bd, cfg, ctx=ctx)
    assert (e["edge_hits"].sum(axis=1) == 100_000).all() and (e["restarts"] == 0).all()
    assert (e["xi"] > 0).all() and (e["xi"] < 1).all() and (e["eta"] > 0).all() and (e["eta"] < 1).all()
    assert ctx.last_stats()["path_steps"] > 6e11
    ij = {(int(round(x * 128)), int(round(y * 128))): k for k, (x, y) in enumerate(zip(px, py))}
    z = []
    for (i, j), k in ij.items():
        q = ij.get((128 - i, j))
        if q is not None and q > k:
            z.append((e["xi"][k] + e["xi"][q] - 1.0) / np.hypot(e["se_xi"][k], e["se_xi"][q]))
    z = np.array(z)
    assert len(z) > 300
    assert np.sum(np.abs(z) > 4) <= 1
    assert 0.5 <= np.mean(z ** 2) <= 1.6  # chi^2 / dof of independent estimates
    # xi increases with x along every horizontal interface line
    for j in (32, 64, 96):
        row = sorted((i, e["xi"][k]) for (i, jj), k in ij.items() if jj == j)
        assert np.all(np.diff([v for _, v in row]) > -4 * 0.5 / np.sqrt(1e5) * np.sqrt(2))


def test_fastmath_accuracy(ctx):
    # performance-mode elementary functions (fastmath.cuh) vs the CUDA library
    import ctypes as C
    m = (C.c_uint64 * 6)()
    sdd._check(sdd.lib().sddg_selftest_fastmath(ctx.handle, C.c_int64(1 << 22), m), ctx.handle)
    exp_u, log_u, sc_u, sqrt_u, rcp_u, log_abs_near1 = list(m)
    assert exp_u <= 4 and log_u <= 4 and sc_u <= 4 and sqrt_u <= 2 and rcp_u <= 2, list(m)
    print("fastmath max ulp (exp, log, sincos, sqrt, rcp, log near 1):", list(m))
    assert log_abs_near1 <= 4096, list(m)  # cancellation near u = 1: <= 1e-12 relative


@pytest.mark.parametrize("kind", [sdd.RING_W, sdd.SHOCK_W, sdd.TWOBUMP_W])
def test_performance_mode_drifts_match_their_definitions(ctx, kind):
    # grad(w)/w from the density's definition (fp64 library) against the fp64
    # table form and the fp32 SFU forms (ring as K q/(1/e + 10), shock with one
    # reciprocal in E = exp(2s), the host-precomputed constants), on 2^22
    # points of the unit square and of a rectangle reaching beyond it (the
    # caps of the exponent arguments), and the fp32 radius argument -2 ln u1
    import ctypes as C

    class Dom(C.Structure):
        _fields_ = [("xmin", C.c_double), ("xmax", C.c_double), ("ymin", C.c_double), ("ymax", C.c_double)]

    fn = sdd.lib().sddg_selftest_drift
    fn.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.POINTER(C.c_double)]
    fn.restype = C.c_int32
    for box in ((0.0, 1.0, 0.0, 1.0), (-2.0, 3.0, -3.0, 4.0)):
        out = (C.c_double * 4)()
        d = Dom(*box)
        sdd._check(fn(ctx.handle, int(kind), C.byref(d), 1 << 22, out), ctx.handle)
        e64, e32, eln, bmax = list(out)
        assert np.isfinite([e64, e32, eln, bmax]).all(), list(out)
        assert bmax > 1.0  # the sample reaches the layer
        assert e64 <= 1e-12 * max(bmax, 1.0), list(out)
        assert e32 <= 2e-5 * max(bmax, 1.0), list(out)
        assert eln <= 5e-5, list(out)  # < 3e-5 from the SFU above d = 2^-8, 2e-8 from the series below
    print("drift self-test", int(kind), list(out))


def test_parity_division_correctly_rounded(ctx):
    # density.cuh div_rn_shared (the parity mode's drift quotients from one
    # shared reciprocal) equals the library's a / b in every bit on 2^28
    # operand pairs, including the quotients just below 1 with the dividend
    # near the top of its binade, where RN(a RN(1/b)) is furthest from a/b
    import ctypes as C
    bad = C.c_uint64(0)
    sdd._check(sdd.lib().sddg_selftest_division(ctx.handle, C.c_int64(1 << 28), C.byref(bad)), ctx.handle)
    assert bad.value == 0


def test_config3_fp32_vs_fp64_exceedances_against_null(ctx):
    # at config 3's 14,273 nodes x 2 fields, count |z| > 4 between
    # independent fp32 and fp64 estimates against the H0 expectation
    # (2 * 14273 * 6.3e-5 = 1.8) and check the aggregate chi^2 / dof
    m = sdd.MonitorFunction.shock(analytic=True)
    spec = sdd.GridSpec(UNIT, 1025, 1025)
    bd = sdd.make_boundary_data(m, spec)
    lay = sdd.build_layout(spec, 8, 8)
    px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("all", 0, m, lay))
    pts = np.stack([px, py], 1)
    a = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd,
                              sdd.WalkConfig(scheme="linear", dt=1e-5, walks=256, seed=101), ctx=ctx)
    b = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd,
                              sdd.WalkConfig(scheme="linear", dt=1e-5, walks=256, seed=202, precision="fp32"),
                              ctx=ctx)
    z = []
    for f, s in (("xi", "se_xi"), ("eta", "se_eta")):
        se = np.hypot(a[s], b[s])
        ok = se > 0
        z.append((a[f][ok] - b[f][ok]) / se[ok])
    z = np.concatenate(z)
    assert len(z) > 20000
    assert np.sum(np.abs(z) > 4) <= 10
    assert 0.9 <= np.mean(z ** 2) <= 1.1


def test_device_api_matches_host_api(ctx):
    # sddg_mc_estimate_batch_device (HBM-resident inputs and records, caller's
    # stream) must give the host-buffer call's records bit for bit
    import torch
    m = sdd.MonitorFunction.ring(analytic=True)
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 65, 65))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=900, seed=9)
    rng = np.random.default_rng(4)
    pts = rng.uniform(0.05, 0.95, (37, 2))
    pid = rng.integers(0, 1 << 47, 37).astype(np.uint64)
    want = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd, cfg, ctx=ctx)
    dev = torch.device("cuda", 0)
    px = torch.tensor(pts[:, 0], dtype=torch.float64, device=dev)
    py = torch.tensor(pts[:, 1], dtype=torch.float64, device=dev)
    tp = torch.tensor(pid.view(np.int64), dtype=torch.int64, device=dev)
    out = torch.zeros(37 * 128, dtype=torch.uint8, device=dev)
    st = torch.cuda.Stream()
    sdd.mc_estimate_batch_device(px, py, tp, out, m, UNIT, bd, cfg, ctx=ctx, stream=st)
    st.synchronize()
    assert out.cpu().numpy().tobytes() == want.tobytes()

"""GPU Perona-Malik (K6) and interface loess (K7) against the reference's
perona_malik / smooth_interface / solve_sdd(smooth_interface) outputs
(tests/golden, made by the reference).  The kernels keep the reference's
operation order; exp/pow come from the CUDA libm (~1 ulp)."""
import numpy as np
import pytest

from paper_1310_3435_b200 import sdd

pytestmark = pytest.mark.gpu
UNIT = sdd.RectDomain(0, 1, 0, 1)


@pytest.mark.parametrize("name,k,steps,scope", [("global", 1000.0, 5, "global"),
                                                ("subdomain", 1000.0, 4, "per_subdomain"),
                                                ("edgestop", 0.5, 6, "global")])
def test_perona_malik_matches_reference(golden, ctx, name, k, steps, scope):
    spec = sdd.GridSpec(UNIT, 33, 33)
    lay = sdd.build_layout(spec, 2, 2)
    dt = float(golden["pm_dt"][0])
    xi, eta, warn = sdd.perona_malik(golden["sdd_running33_xi"], golden["sdd_running33_eta"], spec,
                                     sdd.SmoothConfig(k=k, dt=dt, steps=steps, scope=scope), lay, ctx=ctx)
    want = golden[f"pm_{name}"]
    assert not warn
    assert np.max(np.abs(xi - want[0])) <= 1e-13 and np.max(np.abs(eta - want[1])) <= 1e-13
    # block boundaries held fixed
    X0 = golden["sdd_running33_xi"].reshape(33, 33)
    X = xi.reshape(33, 33)
    assert np.array_equal(X[0], X0[0]) and np.array_equal(X[:, -1], X0[:, -1])
    if scope == "per_subdomain":
        assert np.array_equal(X[16], X0[16]) and np.array_equal(X[:, 16], X0[:, 16])


def test_perona_malik_instability_and_warning(golden, ctx):
    # the reference defaults (dt=1e-4, k=1000) violate hx*hy/4 on fine grids:
    # warning + NumericalError (smoothing.cpp:18-26,115-120)
    spec = sdd.GridSpec(UNIT, 129, 129)
    rng = np.random.default_rng(0)
    X, Y = np.meshgrid(np.linspace(0, 1, 129), np.linspace(0, 1, 129))
    xi = (X + 1e-3 * rng.standard_normal(X.shape)).ravel()
    with pytest.raises(sdd.NumericalError):
        sdd.perona_malik(xi, Y.ravel(), spec, sdd.SmoothConfig(k=1000.0, dt=1e-4, steps=20), ctx=ctx)
    _, _, warn = sdd.perona_malik(xi, Y.ravel(), spec, sdd.SmoothConfig(k=1000.0, dt=1e-4, steps=0), ctx=ctx)
    assert warn


@pytest.mark.parametrize("span", [3, 5, 9])
def test_smooth_interface_matches_reference(golden, ctx, span):
    got = sdd.smooth_interface(golden["loess_in"], span, ctx=ctx)
    assert np.max(np.abs(got - golden[f"loess_{span}"])) <= 1e-13
    assert got[0] == golden["loess_in"][0] and got[-1] == golden["loess_in"][-1]


def test_smooth_interface_is_linear_and_validated(ctx):
    rng = np.random.default_rng(1)
    a, b = rng.random(40), rng.random(40)
    la = sdd.smooth_interface(a, 7, ctx=ctx)
    lb = sdd.smooth_interface(b, 7, ctx=ctx)
    lab = sdd.smooth_interface(2 * a - 3 * b, 7, ctx=ctx)
    assert np.max(np.abs(lab - (2 * la - 3 * lb))) <= 1e-12
    for bad in (2, 4, 41):
        with pytest.raises(sdd.ValidationError):
            sdd.smooth_interface(a, bad, ctx=ctx)


def test_solve_sdd_with_interface_smoothing(golden, ctx):
    m = sdd.MonitorFunction.running_example()
    spec = sdd.GridSpec(UNIT, 33, 33)
    cfg = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=300, seed=2)
    lay = sdd.build_layout(spec, 2, 1)
    plan = sdd.plan_interface_points("all", 0, m, lay)
    r = sdd.solve_sdd(m, lay, plan, cfg, sdd.SolverConfig(tol=1e-12), ctx=ctx,
                      opts=sdd.SddOptions(smooth_interface=True, smooth_span=5))
    want = golden["sdd_smoothed_running33"]
    assert np.max(np.abs(r.xi - want[0])) <= 1e-10 and np.max(np.abs(r.eta - want[1])) <= 1e-10
    # crossing lines: per-line smoothing breaks corner agreement, as in the reference
    lay2 = sdd.build_layout(spec, 2, 2)
    with pytest.raises(sdd.ValidationError, match="corner"):
        sdd.solve_sdd(m, lay2, sdd.plan_interface_points("all", 0, m, lay2), cfg,
                      sdd.SolverConfig(tol=1e-12), ctx=ctx, opts=sdd.SddOptions(smooth_interface=True))

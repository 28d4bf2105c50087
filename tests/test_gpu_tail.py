"""The tail kernel (csrc/walk_tail.cuh): K1 hands the last walks of a batch
to a kernel that runs each on a whole warp.  Every step uses K1's own step,
exit and record functions on the same stream draws, so the results must not
depend on which kernel finished a walk: dumps, estimates, path-steps and
errors are compared bit for bit with K1 alone (SDDG_NO_TAIL=1).  Small dumps
hand nearly every walk over at its 256th step, so the per-path parity tests
against the reference fixtures (test_gpu_walk.py) run through it as well."""
import numpy as np
import pytest

from paper_1310_3435_b200 import sdd

pytestmark = pytest.mark.gpu
UNIT = sdd.RectDomain(0, 1, 0, 1)
FIVE = sdd.RectDomain(-1, 1, -1, 1)


def _both(monkeypatch, fn):
    monkeypatch.delenv("SDDG_NO_TAIL", raising=False)
    a = fn()
    monkeypatch.setenv("SDDG_NO_TAIL", "1")
    b = fn()
    monkeypatch.delenv("SDDG_NO_TAIL", raising=False)
    return a, b


def _table():
    x = np.linspace(0, 1, 33)
    X, Y = np.meshgrid(x, x)
    return sdd.MonitorFunction.tabulated(1.0 + 2.0 * np.exp(-40.0 * ((X - 0.4) ** 2 + (Y - 0.6) ** 2)), UNIT)


CASES = [
    ("ring_fast_linear", lambda: sdd.MonitorFunction.ring(analytic=True), UNIT, "linear", (0.5, 0.5)),
    ("ring_ref_linear", lambda: sdd.MonitorFunction.ring(), UNIT, "linear", (0.5, 0.5)),
    ("shock_fast_linear", lambda: sdd.MonitorFunction.shock(analytic=True), UNIT, "linear", (0.3, 0.45)),
    ("twobump_ref_exp", lambda: sdd.MonitorFunction.two_bump(), UNIT, "exponential", (0.6, 0.4)),
    ("running_ref_exp", lambda: sdd.MonitorFunction.running_example(), UNIT, "exponential", (0.5, 0.5)),
    ("five_ring_fast_exp", lambda: sdd.MonitorFunction.five_ring(analytic=True), FIVE, "exponential", (0.1, 0.2)),
    ("five_ring_ref_linear", lambda: sdd.MonitorFunction.five_ring(), FIVE, "linear", (0.1, 0.2)),
    ("table_ref_linear", _table, UNIT, "linear", (0.45, 0.55)),
    ("table_fast_exp", lambda: _table().with_grad(sdd.GRAD_ANALYTIC), UNIT, "exponential", (0.45, 0.55)),
    ("ring_literal_linear", lambda: sdd.MonitorFunction.ring(analytic=True), UNIT, "literal", (0.5, 0.5)),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_dumps_identical_with_and_without_tail(ctx, monkeypatch, case):
    name, mk, dom, scheme, p = case
    m = mk()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(dom, 33, 33))
    cfg = sdd.WalkConfig(scheme="linear" if scheme == "literal" else scheme, dt=1e-4, lambda_=1000.0, walks=1,
                         seed=11, form="literal" if scheme == "literal" else "reference")
    for n in (700, 4000):  # all walks handed over / handoff once <= 16 per SM remain
        a, b = _both(monkeypatch, lambda: sdd.walk_dump(p, 4242, m, dom, bd, cfg, 0, n, ctx=ctx))
        assert a.tobytes() == b.tobytes(), name
        assert a["steps"].max() > 256  # the long walks did run in the tail kernel


def test_estimates_and_path_steps_identical(ctx, monkeypatch):
    m = sdd.MonitorFunction.ring(analytic=True)
    lay = sdd.build_layout(sdd.GridSpec(UNIT, 65, 65), 2, 2)
    px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("equispaced", 31, m, lay))
    bd = sdd.make_boundary_data(m, lay.global_)
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=3000, seed=3)

    def run():
        e = sdd.mc_estimate_batch(np.stack([px, py], 1), pid, m, UNIT, bd, cfg, ctx=ctx)
        return e, ctx.last_stats()

    (a, sa), (b, sb) = _both(monkeypatch, run)
    assert a.tobytes() == b.tobytes()
    assert sa["path_steps"] == sb["path_steps"] == int(a["path_steps"].sum())
    assert sa["launches"] >= sb["launches"] + 1  # the tail kernel (+ drain rounds)


def test_restarts_in_the_tail(ctx, monkeypatch):
    # max_steps = 300: walks restart on fresh epoch streams, some inside the tail
    m = sdd.MonitorFunction.running_example()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 17, 17))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1, seed=4, max_steps=300)
    a, b = _both(monkeypatch, lambda: sdd.walk_dump((0.5, 0.5), 7, m, UNIT, bd, cfg, 0, 600, ctx=ctx))
    assert a.tobytes() == b.tobytes()
    assert a["epoch"].max() >= 2
    cfg2 = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=600, seed=4, max_steps=300)
    (e1, s1), (e2, s2) = _both(monkeypatch, lambda: (sdd.mc_estimate_batch([(0.5, 0.5)], [7], m, UNIT, bd, cfg2,
                                                                            ctx=ctx), ctx.last_stats()))
    assert e1.tobytes() == e2.tobytes() and s1["path_steps"] == s2["path_steps"]


def test_numerical_error_raised_from_the_tail(ctx, monkeypatch):
    # walks that never exit: 1024 epochs of max_steps, then NumericalError
    m = sdd.MonitorFunction.constant()
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 9, 9))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-9, walks=8, seed=1, max_steps=300)
    monkeypatch.delenv("SDDG_NO_TAIL", raising=False)
    with pytest.raises(sdd.NumericalError):
        sdd.mc_estimate((0.5, 0.5), 1, m, UNIT, bd, cfg, ctx=ctx)


@pytest.mark.parametrize("drain,rounds", [("", 0), ("256,64,32", 3), ("2000", 0)])
def test_drain_rounds_identical(ctx, monkeypatch, drain, rounds):
    # a batch larger than K1's lanes, so its counter runs out while walks are
    # in flight: drain rounds (K1 resumed on its handoffs, repacked) none,
    # three, or a cap above K1's lane count (ignored); estimates, per-node
    # path-steps and the step total unchanged
    m = sdd.MonitorFunction.ring(analytic=True)
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 33, 33))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=50_000, seed=5)
    pts = [(0.45, 0.5), (0.5, 0.2), (0.3, 0.7), (0.6, 0.6)]
    monkeypatch.setenv("SDDG_NO_TAIL", "1")
    ref = sdd.mc_estimate_batch(pts, [1, 2, 3, 4], m, UNIT, bd, cfg, ctx=ctx)
    s_ref = ctx.last_stats()
    monkeypatch.delenv("SDDG_NO_TAIL")
    monkeypatch.setenv("SDDG_DRAIN", drain)
    e = sdd.mc_estimate_batch(pts, [1, 2, 3, 4], m, UNIT, bd, cfg, ctx=ctx)
    st = ctx.last_stats()
    assert e.tobytes() == ref.tobytes()
    assert st["path_steps"] == s_ref["path_steps"]
    assert st["launches"] == s_ref["launches"] + 1 + 2 * rounds
    assert st["tail_handoffs"] > 0

"""Multi-GPU contexts of the C-ABI (csrc/team.cu) on the one B200 of a test
box: the sharded path must be bit-identical to a single-device context.

* sddg_create_dist with one rank: the NCCL exchange (ncclCommInitRank +
  in-place ncclAllGather of the 128-B records) over a one-rank communicator;
* sddg_create_multi with device 0 listed 2-3 times: several independent
  ranks driven from one process (one host thread each).  By default the
  exchange is fused into K2 (each member's reduce kernel stores its records
  into the owner's output, as over NVLink peer memory); with SDDG_TEAM_COPY=1
  the members pack, copy and scatter as the NCCL fallback does -- every shard
  boundary, the pack/scatter kernels and the subdomain ranges run exactly as
  on several GPUs, without any kernel waiting on another (
  B200_PROFILING.md on single-GPU stand-ins).
* the cost model behind the shards against measured per-node path-steps.
"""
import numpy as np
import pytest

from paper_1310_3435_b200 import sdd

pytestmark = pytest.mark.gpu
UNIT = sdd.RectDomain(0, 1, 0, 1)


@pytest.fixture(scope="module")
def dist1():
    c = sdd.Context.dist(0, 0, 1, sdd.nccl_unique_id())
    yield c
    c.close()


@pytest.fixture(scope="module")
def multi3():
    c = sdd.Context.multi([0, 0, 0])
    yield c
    c.close()


@pytest.fixture(scope="module")
def multi3copy():
    import os
    os.environ["SDDG_TEAM_COPY"] = "1"  # read when the context is made
    try:
        c = sdd.Context.multi([0, 0, 0])
    finally:
        del os.environ["SDDG_TEAM_COPY"]
    yield c
    c.close()


def _config2_sample(k=90):
    m = sdd.MonitorFunction.ring(analytic=True)
    spec = sdd.GridSpec(UNIT, 129, 129)
    lay = sdd.build_layout(spec, 4, 4)
    px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("all", 0, m, lay))
    s = np.linspace(0, len(px) - 1, k).round().astype(int)
    return m, spec, np.stack([px[s], py[s]], 1), pid[s]


def test_team_info(ctx, dist1, multi3):
    assert ctx.team_info() == {"rank": 0, "nranks": 1, "local_devices": 1, "nccl": False}
    assert dist1.team_info() == {"rank": 0, "nranks": 1, "local_devices": 1, "nccl": True}
    assert multi3.team_info() == {"rank": 0, "nranks": 3, "local_devices": 3, "nccl": False}


@pytest.mark.parametrize("which", ["dist1", "multi3", "multi3copy"])
def test_sharded_estimates_bit_identical(ctx, request, which):
    team = request.getfixturevalue(which)
    m, spec, pts, pid = _config2_sample()
    bd = sdd.make_boundary_data(m, spec)
    for cfg in (sdd.WalkConfig(scheme="linear", dt=2e-5, walks=700, seed=3),
                sdd.WalkConfig(scheme="linear", dt=2e-5, walks=700, seed=3, precision="fp32")):
        want = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd, cfg, ctx=ctx)
        got = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd, cfg, ctx=team)
        assert got.tobytes() == want.tobytes()
        assert team.last_stats()["path_steps"] == int(want["path_steps"].sum())
    # reference (FD) drift, exponential scheme
    mr = sdd.MonitorFunction.ring()
    cfg = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=300, seed=5)
    assert (sdd.mc_estimate_batch(pts[:20], pid[:20], mr, UNIT, bd, cfg, ctx=team).tobytes() ==
            sdd.mc_estimate_batch(pts[:20], pid[:20], mr, UNIT, bd, cfg, ctx=ctx).tobytes())


def test_sharded_device_api_bit_identical(ctx, dist1, multi3):
    import torch
    m, spec, pts, pid = _config2_sample(40)
    bd = sdd.make_boundary_data(m, spec)
    cfg = sdd.WalkConfig(scheme="linear", dt=2e-5, walks=500, seed=8)
    want = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd, cfg, ctx=ctx)
    dev = torch.device("cuda", 0)
    px = torch.tensor(pts[:, 0], dtype=torch.float64, device=dev)
    py = torch.tensor(pts[:, 1], dtype=torch.float64, device=dev)
    tp = torch.tensor(pid.view(np.int64), dtype=torch.int64, device=dev)
    for team in (dist1, multi3):
        out = torch.zeros(len(pid) * 128, dtype=torch.uint8, device=dev)
        st = torch.cuda.Stream()
        sdd.mc_estimate_batch_device(px, py, tp, out, m, UNIT, bd, cfg, ctx=team, stream=st)
        st.synchronize()
        assert out.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("which", ["dist1", "multi3", "multi3copy"])
def test_sharded_solve_sdd_bit_identical(ctx, request, which):
    team = request.getfixturevalue(which)
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 65, 65)
    lay = sdd.build_layout(spec, 4, 2)  # 8 subdomains over 3 ranks: ranges 2, 3, 3
    plan = sdd.plan_interface_points("equispaced", 15, m, lay)
    wcfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=400, seed=1)
    scfg = sdd.SolverConfig(tol=1e-12, method="rbsor")
    a = sdd.solve_sdd(m, lay, plan, wcfg, scfg, ctx=ctx)
    b = sdd.solve_sdd(m, lay, plan, wcfg, scfg, ctx=team)
    assert np.array_equal(a.xi, b.xi) and np.array_equal(a.eta, b.eta)
    assert (a.mc_points, a.restarts, a.path_steps, a.warnings) == (b.mc_points, b.restarts, b.path_steps,
                                                                   b.warnings)
    bd = sdd.make_boundary_data(m, spec)
    ia = sdd.solve_interfaces(plan, m, bd, wcfg, lay, ctx=ctx)
    ib = sdd.solve_interfaces(plan, m, bd, wcfg, lay, ctx=team)
    for u, v in zip(ia.xi + ia.eta + ia.se_xi, ib.xi + ib.eta + ib.se_xi):
        assert np.array_equal(u, v)
    sa = sdd.stochastic_full(m, sdd.GridSpec(UNIT, 17, 17), sdd.WalkConfig(walks=200, seed=2), ctx=ctx)
    sb = sdd.stochastic_full(m, sdd.GridSpec(UNIT, 17, 17), sdd.WalkConfig(walks=200, seed=2), ctx=team)
    assert np.array_equal(sa[0], sb[0]) and np.array_equal(sa[1], sb[1])


def test_cost_model_predicts_measured_path_steps(ctx):
    # The shard plan balances predicted cost; what matters is the measured
    # work.  Per-node path-steps measured by K1 against the exit-time model,
    # and the imbalance of the measured steps over 8 ranks under the plan.
    report = {}
    cases = [("config2_ring", sdd.MonitorFunction.ring(analytic=True), 129, 4, 2e-5, 2000, "fp64"),
             ("config3_shock", sdd.MonitorFunction.shock(analytic=True), 1025, 8, 1e-5, 64, "fp32")]
    for name, m, n, s, dt, walks, prec in cases:
        spec = sdd.GridSpec(UNIT, n, n)
        lay = sdd.build_layout(spec, s, s)
        px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("all", 0, m, lay))
        pts = np.stack([px, py], 1)
        cfg = sdd.WalkConfig(scheme="linear", dt=dt, walks=walks, seed=1, precision=prec)
        bd = sdd.make_boundary_data(m, spec)
        e = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd, cfg, ctx=ctx)
        rank, cost = sdd.shard_plan(pts, m, UNIT, cfg, 8)
        meas = e["path_steps"].astype(np.float64)
        corr = float(np.corrcoef(cost, meas)[0, 1])
        ratio = float(meas.sum() / cost.sum())
        loads = np.array([meas[rank == r].sum() for r in range(8)])
        imb = float(loads.max() / loads.mean() - 1)
        report[name] = {"nodes": len(px), "corr": corr, "measured_over_predicted": ratio,
                        "measured_imbalance_8_ranks": imb}
        assert corr > 0.95, report
        assert 0.7 < ratio < 1.3, report
        assert imb < 0.03, report
    print("cost model vs measured path-steps:", report)

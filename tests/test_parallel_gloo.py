"""Multi-rank host logic of the sharded SDD path on CPU (gloo, world size 2
and 3): node sharding, the all-gather of estimate records, interface fill
and subdomain assembly must equal the single-process result bit for bit.
Walk and solver kernels are replaced by deterministic stand-ins here (the
GPU kernels are covered by the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1310_3435_b200 import parallel, sdd

UNIT = sdd.RectDomain(0, 1, 0, 1)


def fake_estimator(px, py, pid):
    out = np.zeros(len(px), sdd.ESTIMATE_DTYPE)
    out["xi"] = px + 0.01 * np.sin(7 * py)
    out["eta"] = py + 0.01 * np.cos(5 * px)
    out["se_xi"] = 1e-3 * px
    out["se_eta"] = 1e-3 * py
    out["walks"] = 100
    out["restarts"] = (np.asarray(pid) % 3 == 0).astype(np.int64)
    out["edge_hits"][:, 0] = 100
    return out


def fake_solver_factory(layout):
    def solver(lo, hi):
        by, bx = layout.block_y + 1, layout.block_x + 1
        f = np.zeros((hi - lo, 2, by, bx))
        for k, s in enumerate(range(lo, hi)):
            f[k, 0] = s + np.arange(bx)[None, :] / bx
            f[k, 1] = -s - np.arange(by)[:, None] / by
        return f
    return solver


def _problem():
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 33, 33)
    lay = sdd.build_layout(spec, 4, 2)
    plan = sdd.plan_interface_points("equispaced", 9, m, lay)
    return m, spec, lay, plan


def _worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        m, spec, lay, plan = _problem()
        bd = sdd.make_boundary_data(m, spec)
        cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=100, seed=1)
        ifc, est = parallel.solve_interfaces_distributed(plan, m, bd, cfg, lay, estimator=fake_estimator)
        px, py, pid = sdd.interface_nodes(m, lay, plan)
        ref = sdd.fill_interfaces(m, lay, plan, bd, fake_estimator(px, py, pid))
        assert est.tobytes() == fake_estimator(px, py, pid).tobytes()
        for a, b in zip(ifc.xi + ifc.eta + ifc.se_xi, ref.xi + ref.eta + ref.se_xi):
            assert np.array_equal(a, b)
        assert ifc.restarts == ref.restarts
        xi, eta, _, _ = parallel.solve_sdd_distributed(m, lay, plan, cfg, sdd.SolverConfig(),
                                                       estimator=fake_estimator,
                                                       solver=fake_solver_factory(lay))
        rxi, reta = sdd.assemble(lay, fake_solver_factory(lay)(0, lay.subdomain_count()))
        assert np.array_equal(xi, rxi) and np.array_equal(eta, reta)
        for kw in ({"transport": "bogus"}, {"transport": "peer", "estimator": fake_estimator}):
            try:
                parallel.solve_interfaces_distributed(plan, m, bd, cfg, lay, **kw)
            except sdd.ValidationError:
                pass
            else:
                raise AssertionError(f"{kw} accepted")
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as exc:  # surface the failure in the parent
        errq.put(f"rank {rank}: {type(exc).__name__}: {exc}")
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_interfaces_and_assembly_match_single_process(world):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(world, _free_port(), errq), nprocs=world, join=True,
                       start_method="spawn")
    assert errq.empty(), errq.get()


def test_shard_covers_each_node_once_and_balances():
    rng = np.random.default_rng(0)
    costs = rng.random(1000) ** 3
    parts = parallel.shard(costs, 8)
    allidx = np.sort(np.concatenate(parts))
    assert np.array_equal(allidx, np.arange(1000))
    loads = [costs[p].sum() for p in parts]
    assert max(loads) / min(loads) < 1.02


def test_subdomain_ranges_partition():
    for n, w in [(64, 8), (16, 3), (4, 8)]:
        r = [parallel.subdomain_range(n, w, k) for k in range(w)]
        assert r[0][0] == 0 and r[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))


def test_config3_node_count_and_cost_order():
    spec = sdd.GridSpec(UNIT, 1025, 1025)
    lay = sdd.build_layout(spec, 8, 8)
    m = sdd.MonitorFunction.shock(analytic=True)
    plan = sdd.plan_interface_points("all", 0, m, lay)
    px, py, pid = sdd.interface_nodes(m, lay, plan)
    assert len(px) == 14273 and len(np.unique(pid)) == 14273
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-5, walks=1_000_000, seed=1, precision="fp32")
    rank, cost = sdd.shard_plan(np.stack([px, py], 1), m, UNIT, cfg, 8)
    loads = [cost[rank == r].sum() for r in range(8)]
    assert max(loads) / min(loads) < 1.001
    # the torch.distributed driver shards exactly like the C-ABI plan
    parts = parallel.node_shards(px, py, m, UNIT, cfg, 8)
    assert all(np.array_equal(parts[r], np.nonzero(rank == r)[0]) for r in range(8))
    # and the rule is parallel.shard's LPT
    ref = parallel.shard(cost, 8)
    assert all(np.array_equal(parts[r], ref[r]) for r in range(8))

"""Fused finalize + gather (sddg_mc_estimate_gather): K2 stores every
record straight into each rank's gather buffer (CUDA IPC peer memory).

* one process, two local buffers: the fused stores land at the global
  slots, byte-identical to sddg_mc_estimate_batch;
* two processes on one GPU (gloo for the host handshake only; no kernel
  waits on another): transport="peer" of the sharded interface solve
  equals the single-process result bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1310_3435_b200 import parallel, sdd

pytestmark = pytest.mark.gpu
UNIT = sdd.RectDomain(0, 1, 0, 1)


def _problem():
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 33, 33)
    lay = sdd.build_layout(spec, 4, 2)
    plan = sdd.plan_interface_points("equispaced", 9, m, lay)
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1500, seed=11)
    return m, spec, lay, plan, cfg


def test_fused_gather_local_buffers(ctx):
    m, spec, lay, plan, cfg = _problem()
    bd = sdd.make_boundary_data(m, spec)
    px, py, pid = sdd.interface_nodes(m, lay, plan)
    want = sdd.mc_estimate_batch(np.stack([px, py], 1), pid, m, UNIT, bd, cfg, ctx=ctx)
    a, b = sdd.PeerGather(len(px), ctx), sdd.PeerGather(len(px), ctx)
    try:
        # two disjoint halves, in scrambled order, each landing at its global slot
        order = np.random.default_rng(3).permutation(len(px))
        for part in (order[: len(px) // 2], order[len(px) // 2:]):
            sdd.mc_estimate_gather(np.stack([px[part], py[part]], 1), pid[part], part,
                                   [a.ptr.value, b.ptr.value], len(px), m, UNIT, bd, cfg, ctx=ctx)
        assert a.read().tobytes() == want.tobytes()
        assert b.read().tobytes() == want.tobytes()
        with pytest.raises(sdd.ValidationError):
            sdd.mc_estimate_gather([[0.5, 0.5]], [1], [len(px)], [a.ptr.value], len(px), m, UNIT, bd,
                                   cfg, ctx=ctx)
    finally:
        a.close()
        b.close()


def _worker(rank, world, port, errq, want_bytes):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ctx = sdd.Context(0)
        m, spec, lay, plan, cfg = _problem()
        bd = sdd.make_boundary_data(m, spec)
        ifc, est = parallel.solve_interfaces_distributed(plan, m, bd, cfg, lay, ctx=ctx,
                                                         transport="peer")
        assert est.tobytes() == want_bytes
        dist.barrier()
        dist.destroy_process_group()
        ctx.close()
    except BaseException as exc:
        errq.put(f"rank {rank}: {type(exc).__name__}: {exc}")
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_peer_transport_two_processes_bit_identical(ctx):
    m, spec, lay, plan, cfg = _problem()
    bd = sdd.make_boundary_data(m, spec)
    px, py, pid = sdd.interface_nodes(m, lay, plan)
    want = sdd.mc_estimate_batch(np.stack([px, py], 1), pid, m, UNIT, bd, cfg, ctx=ctx)
    mpc = mp.get_context("spawn")
    errq = mpc.SimpleQueue()
    mp.start_processes(_worker, args=(2, _free_port(), errq, want.tobytes()), nprocs=2, join=True,
                       start_method="spawn")
    assert errq.empty(), errq.get()

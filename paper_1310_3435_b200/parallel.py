"""Multi-GPU sharding of the SDD hot path (one process per GPU,
torch.distributed: NCCL over NVLink on the B200 box, gloo on CPU).

The reference parallelises with a std::thread pool over interface points and
over subdomains (proj/src/decomposition.cpp:172-174, 298-355).
Here every rank
  1. walks a cost-balanced shard of the interface nodes (K1/K2 on its GPU),
  2. all-gathers the fixed-size sddg_estimate records (the one data-path
     collective: ~128 B per node, 1.8 MB for config 3's 14,273 nodes) --
     transport="nccl" through torch.distributed, transport="peer" fused
     into the finalize kernel K2, which stores every record straight into
     each rank's gather buffer over NVLink peer memory (CUDA IPC),
  3. fills the interface lines (identical on every rank, host C++),
  4. solves a contiguous range of subdomains (K3 on its GPU),
  5. all-gathers the subdomain fields and assembles the mesh.
Estimates are a pure function of (seed, point_id, walk) and each node is
reduced on one rank in the reference's chunk order, so the result is
bit-identical for any world size.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import sdd


def node_shards(px, py, m: sdd.MonitorFunction, domain: sdd.RectDomain, cfg: sdd.WalkConfig, world: int):
    """The node shards of the C-ABI's multi-GPU contexts (sddg_shard_plan:
    expected path-steps from the walk's exit-time model, LPT over ranks), so
    this torch.distributed driver and sddg_create_dist shard identically.
    Returns a list of sorted index arrays, one per rank."""
    rank_of, _ = sdd.shard_plan(np.stack([px, py], 1), m, domain, cfg, world)
    return [np.nonzero(rank_of == r)[0] for r in range(world)]


def shard(costs, world: int):
    """Greedy LPT assignment of items to `world` ranks (the rule of
    sddg_shard_plan); deterministic.
    Returns a list of sorted index arrays, one per rank."""
    costs = np.asarray(costs, dtype=np.float64)
    order = np.argsort(-costs, kind="stable")
    load = np.zeros(world)
    owner = np.empty(len(costs), np.int64)
    for i in order:
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += costs[i]
    return [np.nonzero(owner == r)[0] for r in range(world)]


def _comm_device():
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def all_gather_rows(local: np.ndarray, indices: np.ndarray, n_total: int, row_bytes: int):
    """All-gather variable-size shards of fixed-size binary rows back into
    global order.  local: uint8-viewable array of len(indices) rows."""
    world = dist.get_world_size()
    dev = _comm_device()
    counts = torch.tensor([len(indices)], dtype=torch.int64, device=dev)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts)
    cap = int(max(int(c.item()) for c in all_counts))
    buf = np.zeros((cap, row_bytes), np.uint8)
    if len(indices):
        buf[:len(indices)] = np.ascontiguousarray(local).view(np.uint8).reshape(len(indices), row_bytes)
    idx = np.full(cap, -1, np.int64)
    idx[:len(indices)] = indices
    t_rows = torch.from_numpy(buf).to(dev)
    t_idx = torch.from_numpy(idx).to(dev)
    g_rows = torch.empty((world * cap, row_bytes), dtype=torch.uint8, device=dev)
    g_idx = torch.empty(world * cap, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(g_rows, t_rows)
    dist.all_gather_into_tensor(g_idx, t_idx)
    g_rows, g_idx = g_rows.cpu().numpy(), g_idx.cpu().numpy()
    out = np.zeros((n_total, row_bytes), np.uint8)
    ok = g_idx >= 0
    out[g_idx[ok]] = g_rows[ok]
    return out


def peer_gather_estimates(px, py, pid, mine, m, domain, bd, cfg, ctx=None):
    """Walk this rank's nodes and deliver every record to every rank with
    the fused K2 + peer-store path (sddg_mc_estimate_gather).  The handles
    travel once over the host group; afterwards no collective runs on the
    data path, only the completion barrier."""
    rank, world = dist.get_rank(), dist.get_world_size()
    n_total = len(px)
    buf = sdd.PeerGather(n_total, ctx)
    try:
        handles = [None] * world
        dist.all_gather_object(handles, buf.handle)
        ptrs = [buf.ptr.value if r == rank else buf.open(handles[r]) for r in range(world)]
        if len(mine):
            sdd.mc_estimate_gather(np.stack([px[mine], py[mine]], 1), pid[mine], mine, ptrs, n_total,
                                   m, domain, bd, cfg, ctx=ctx)
        dist.barrier()          # every rank's stores into every buffer have completed
        est = buf.read()
        dist.barrier()          # nobody frees a buffer a peer may still map
    finally:
        buf.close()
    return est


def solve_interfaces_distributed(plan, m, bd, cfg, layout, estimator=None, ctx=None, interp="linear",
                                 transport="nccl"):
    """solve_interfaces over all ranks.  estimator(px, py, pid) -> records
    (sdd.ESTIMATE_DTYPE); default: this rank's GPU through the C-ABI.
    transport="peer" uses the fused K2 peer-store gather instead of the
    NCCL all-gather (needs the default estimator)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    px, py, pid = sdd.interface_nodes(m, layout, plan)
    mine = node_shards(px, py, m, layout.global_.domain, cfg, world)[rank]
    if transport == "peer":
        if estimator is not None:
            raise sdd.ValidationError("transport='peer' runs the walks itself; no estimator")
        est = peer_gather_estimates(px, py, pid, mine, m, layout.global_.domain, bd, cfg, ctx)
        return sdd.fill_interfaces(m, layout, plan, bd, est, interp=interp), est
    if transport != "nccl":
        raise sdd.ValidationError(f"unknown transport {transport!r}")
    if estimator is None:
        def estimator(x, y, p):
            return sdd.mc_estimate_batch(np.stack([x, y], 1), p, m, layout.global_.domain, bd, cfg,
                                         ctx=ctx)
    local = estimator(px[mine], py[mine], pid[mine]) if len(mine) else np.zeros(0, sdd.ESTIMATE_DTYPE)
    rows = all_gather_rows(local, mine, len(px), sdd.ESTIMATE_DTYPE.itemsize)
    est = rows.view(sdd.ESTIMATE_DTYPE).reshape(-1)
    return sdd.fill_interfaces(m, layout, plan, bd, est, interp=interp), est


def subdomain_range(n_sub: int, world: int, rank: int):
    lo = (n_sub * rank) // world
    return lo, (n_sub * (rank + 1)) // world


def solve_sdd_distributed(m, layout, plan, wcfg, scfg, bc_mode=sdd.BC_REFERENCE, estimator=None,
                          solver=None, ctx=None, interp="linear", transport="nccl"):
    """solve_sdd over all ranks; every rank returns the assembled (xi, eta)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    bd = sdd.make_boundary_data(m, layout.global_, bc_mode)
    ifc, est = solve_interfaces_distributed(plan, m, bd, wcfg, layout, estimator, ctx, interp,
                                            transport)
    n_sub = layout.subdomain_count()
    lo, hi = subdomain_range(n_sub, world, rank)
    if solver is None:
        def solver(a, b):
            return sdd.solve_subdomains(m, layout, ifc.xi, ifc.eta, scfg, a, b, bc_mode, ctx)[0]
    local = solver(lo, hi)
    bx, by = layout.block_x + 1, layout.block_y + 1
    rows = all_gather_rows(np.ascontiguousarray(local, dtype=np.float64), np.arange(lo, hi), n_sub,
                           2 * bx * by * 8)
    fields = rows.view(np.float64).reshape(n_sub, 2, by, bx)
    xi, eta = sdd.assemble(layout, fields)
    return xi, eta, ifc, est

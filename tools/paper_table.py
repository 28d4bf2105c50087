"""The reference's own end-to-end workload on one B200 next to the reference
CPU build: the paper's timing table
as the reference's acceptance criterion c11 runs it
(proj/tests/acceptance.cpp:331-372): five-ring density on [-1,1]^2, 4x4
subdomains, optimal interface placement, exponential time stepping
(lambda 1000), N = 5000 walks per node, seed 1, default SolverConfig
(reference Jacobi, tol 1e-8), grids 37^2 ... 197^2.

Per grid: T_stoc / T_sub / T_total of solve_sdd and T_1 of the single-domain
solve, ours (sddg_solve_sdd, GPU: reference-mode drift with the reference
Jacobi or RB-SOR, and the performance-mode five-ring drift with RB-SOR) and the
reference's (oracle/_ref on every
host thread; T_1 sequential as in c11), plus the largest difference between
the two meshes (same streams, reference-mode drift: libm ulps only).

usage: python tools/paper_table.py [--grids 37,77,157] [--no-ref-t1-above N]
Prints one JSON object (copied into profiles/ per round)."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1310_3435_b200 import sdd  # noqa: E402
from oracle import bindings as B  # noqa: E402  (the reference CPU arm: timing + mesh check)


def ours(m, n, ctx, solver):
    spec = sdd.GridSpec(m.domain, n, n)
    lay = sdd.build_layout(spec, 4, 4)
    plan = sdd.plan_interface_points("optimal", 0, m, lay)
    cfg = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=5000, seed=1)
    scfg = sdd.SolverConfig(tol=1e-8, method=solver)
    sdd.solve_sdd(m, lay, plan, cfg, scfg, ctx=ctx)  # warm-up (module load, buffers)
    t0 = time.perf_counter()
    r = sdd.solve_sdd(m, lay, plan, cfg, scfg, ctx=ctx)
    wall = time.perf_counter() - t0
    lay1 = sdd.build_layout(spec, 1, 1)
    plan1 = sdd.plan_interface_points("all", 0, m, lay1)
    t0 = time.perf_counter()
    single = sdd.solve_sdd(m, lay1, plan1, sdd.WalkConfig(walks=1), scfg, ctx=ctx)
    t_1 = time.perf_counter() - t0
    mesh = sdd.invert_mesh(r.xi, r.eta, spec, n, n, ctx=ctx)
    ref = sdd.invert_mesh(single.xi, single.eta, spec, n, n, ctx=ctx)
    q = sdd.quality_report(mesh, ref, m, ctx=ctx)
    return r, {"t_stoc_s": r.t_stoc, "t_sub_s": r.t_sub, "t_total_s": r.t_stoc + r.t_sub + r.t_smooth,
               "wall_s": wall, "t_1_s": t_1, "mc_points": r.mc_points, "path_steps": r.path_steps,
               "path_steps_per_s": r.path_steps / r.t_stoc if r.t_stoc > 0 else None,
               "r_mean": q.r_mean, "q_max": q.q_max, "solver": solver}


def reference(n, threads, with_t1):
    ref = B.Ref()
    dens, dom = B.density(B.FIVE_RING), B.Domain(-1.0, 1.0, -1.0, 1.0)
    cfg = B.walk_cfg(scheme="exponential", lam=1000.0, walks=5000, seed=1)
    xi, eta, t = ref.solve_sdd(dens, dom, n, n, 4, 4, 2, 0, cfg, tol=1e-8, threads=threads)
    out = {"t_stoc_s": t[0], "t_sub_s": t[1], "t_total_s": float(t.sum()), "threads": threads}
    if with_t1:
        t0 = time.perf_counter()
        ref.solve_single_domain(dens, dom, n, n, tol=1e-8)
        out["t_1_s"] = time.perf_counter() - t0
    return xi, eta, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grids", default="37,77,117,157,197")
    ap.add_argument("--no-ref", action="store_true")
    ap.add_argument("--ref-t1-max", type=int, default=157, help="largest grid for the reference T_1")
    args = ap.parse_args()
    ctx = sdd.Context(0)
    m = sdd.MonitorFunction.five_ring()
    m_fast = sdd.MonitorFunction.five_ring(analytic=True)  # performance-mode drift
    threads = os.cpu_count() or 1
    rows = {}
    for n in (int(g) for g in args.grids.split(",")):
        r, row = ours(m, n, ctx, "jacobi")
        _, row_sor = ours(m, n, ctx, "rbsor")
        rf, row_fast = ours(m_fast, n, ctx, "rbsor")
        rows[n] = {"ours": row, "ours_rbsor": row_sor, "ours_fast_rbsor": row_fast}
        if not args.no_ref:
            xi, eta, rr = reference(n, threads, n <= args.ref_t1_max)
            rows[n]["reference_cpu"] = rr
            rows[n]["max_abs_mesh_diff"] = float(max(np.max(np.abs(xi - r.xi)), np.max(np.abs(eta - r.eta))))
            rows[n]["max_abs_mesh_diff_fast"] = float(max(np.max(np.abs(xi - rf.xi)),
                                                          np.max(np.abs(eta - rf.eta))))
            rows[n]["t_total_speedup"] = rr["t_total_s"] / row["t_total_s"]
            rows[n]["t_total_speedup_fast"] = rr["t_total_s"] / row_fast["t_total_s"]
        print(n, json.dumps(rows[n]), file=sys.stderr, flush=True)
    print(json.dumps({"workload": "paper table / acceptance c11: five-ring on [-1,1]^2, 4x4, optimal placement, "
                      "exponential lambda 1000, N 5000, seed 1, tol 1e-8", "gpu": ctx.device_name()
                      if hasattr(ctx, "device_name") else "cuda:0", "host_threads": threads,
                      "grids": rows}, indent=1))


if __name__ == "__main__":
    main()

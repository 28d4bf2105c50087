"""Throughput of the BASELINE.json configs on one B200 (run under gpurun).
Prints one JSON object; copied into profiles/ per round."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
out = {}


def walk_rate(m, pts, pids, bd, cfg, reps=2):
    sdd.mc_estimate_batch(pts[:8], pids[:8], m, UNIT, bd, cfg, ctx=ctx)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        sdd.mc_estimate_batch(pts, pids, m, UNIT, bd, cfg, ctx=ctx)
        wall = time.perf_counter() - t0
        st = ctx.last_stats()
        r = {"path_steps": st["path_steps"], "k1_ms": st["kernel_ms"], "wall_s": wall,
             "path_steps_per_s": st["path_steps"] / (st["kernel_ms"] / 1e3)}
        best = r if best is None or r["path_steps_per_s"] > best["path_steps_per_s"] else best
    return best


def nodes_of(grid, subs, place="all", k=0, m=None):
    lay = sdd.build_layout(sdd.GridSpec(UNIT, grid, grid), subs, subs)
    plan = sdd.plan_interface_points(place, k, m or sdd.MonitorFunction.ring(), lay)
    px, py, pid = sdd.interface_nodes(m or sdd.MonitorFunction.ring(), lay, plan)
    return lay, plan, np.stack([px, py], 1), pid


# ---- config 1 (full): 65^2, 2x2, equispaced(31), ring, dt 1e-4, 1e4 paths, fp64
for mode in ("reference_fd", "analytic"):
    m = sdd.MonitorFunction.ring(analytic=mode == "analytic")
    lay, plan, pts, pid = nodes_of(65, 2, "equispaced", 31, m)
    bd = sdd.make_boundary_data(m, lay.global_)
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=10_000, seed=1)
    out[f"config1_walks_{mode}"] = walk_rate(m, pts, pid, bd, cfg)
    r = sdd.solve_sdd(m, lay, plan, cfg, sdd.SolverConfig(tol=1e-10), ctx=ctx)
    out[f"config1_solve_sdd_{mode}"] = {"t_stoc_s": r.t_stoc, "t_sub_s": r.t_sub, "mc_points": r.mc_points,
                                        "path_steps": r.path_steps, "solver": "jacobi (reference iteration) tol 1e-10"}

# ---- config 2 walk phase in reference (FD) mode, 1e4 of the 1e5 paths
m = sdd.MonitorFunction.ring()
lay, plan, pts, pid = nodes_of(129, 4, m=m)
bd = sdd.make_boundary_data(m, lay.global_)
out["config2_walks_reference_fd_1e4"] = walk_rate(m, pts, pid, bd,
                                                  sdd.WalkConfig(scheme="linear", dt=2e-5, walks=10_000, seed=1), reps=1)

# ---- config 3: 1025^2, 8x8, shock, dt 1e-5, fp32 walks (fp64 sums), 1e4 of 1e6 paths
m = sdd.MonitorFunction.shock(analytic=True)
lay, plan, pts, pid = nodes_of(1025, 8, m=m)
bd = sdd.make_boundary_data(m, lay.global_)
for prec in ("fp32", "fp64"):
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-5, walks=10_000 if prec == "fp32" else 2_000, seed=1,
                         precision=prec)
    r = walk_rate(m, pts, pid, bd, cfg, reps=1)
    r["paths_per_node"] = cfg.walks
    r["full_config_s_est"] = r["k1_ms"] / 1e3 * (1_000_000 / cfg.walks)
    out[f"config3_walks_{prec}"] = r

# ---- config 5: 4096 uniform start points (numpy seed 1), ring, dt 1e-5
rng = np.random.default_rng(1)
p5 = rng.uniform(0.0, 1.0, size=(4096, 2))
p5 = np.clip(p5, 1e-9, 1 - 1e-9)
pid5 = np.arange(4096, dtype=np.uint64)
bd5 = sdd.make_boundary_data(sdd.MonitorFunction.ring(), sdd.GridSpec(UNIT, 129, 129), sdd.BC_IDENTITY)
for prec in ("fp64", "fp32"):
    for walks in (1_000, 10_000, 100_000):
        if prec == "fp64" and walks == 100_000:
            continue
        cfg = sdd.WalkConfig(scheme="linear", dt=1e-5, walks=walks, seed=1, precision=prec)
        out[f"config5_{prec}_{walks}"] = walk_rate(sdd.MonitorFunction.ring(analytic=True), p5, pid5, bd5, cfg,
                                                   reps=1)

# ---- config 4 end to end: 513^2, 4x4, two-bump, 32 integral-w-equidistributed nodes per
# line, 2e5 paths, dt 1e-5 fp64, spline fill, Laplacian smoothing (5 sweeps), quality
# against the single-domain solve -- all on the GPU
import time as _t
m4 = sdd.MonitorFunction.two_bump(analytic=True)
spec4 = sdd.GridSpec(UNIT, 513, 513)
lay4 = sdd.build_layout(spec4, 4, 4)
plan4 = sdd.plan_interface_points("equidistributed", 32, m4, lay4)
# warm-up call (module loading of every kernel on the path), then the timed one
sdd.solve_sdd(m4, lay4, plan4, sdd.WalkConfig(scheme="linear", dt=1e-5, walks=2_000, seed=2),
              sdd.SolverConfig(tol=1e-10, method="rbsor"), ctx=ctx, opts=sdd.SddOptions(interp="spline"))
sdd.solve_sdd(m4, sdd.build_layout(spec4, 1, 1), sdd.plan_interface_points("all", 0, m4, sdd.build_layout(spec4, 1, 1)),
              sdd.WalkConfig(walks=1), sdd.SolverConfig(tol=1e-6, method="rbsor"), ctx=ctx)
t0 = _t.perf_counter()
r4 = sdd.solve_sdd(m4, lay4, plan4, sdd.WalkConfig(scheme="linear", dt=1e-5, walks=200_000, seed=1),
                   sdd.SolverConfig(tol=1e-10, method="rbsor"), ctx=ctx, opts=sdd.SddOptions(interp="spline"))
t_sdd = _t.perf_counter() - t0
t0 = _t.perf_counter()
xs, es = sdd.laplacian_smooth(r4.xi, r4.eta, spec4, 5, ctx=ctx)
t_smooth = _t.perf_counter() - t0
mesh4 = sdd.invert_mesh(xs, es, spec4, 513, 513, ctx=ctx)
t0 = _t.perf_counter()
lay1 = sdd.build_layout(spec4, 1, 1)
single = sdd.solve_sdd(m4, lay1, sdd.plan_interface_points("all", 0, m4, lay1), sdd.WalkConfig(walks=1),
                       sdd.SolverConfig(tol=1e-10, method="rbsor"), ctx=ctx)
t_1 = _t.perf_counter() - t0
ref4 = sdd.invert_mesh(single.xi, single.eta, spec4, 513, 513, ctx=ctx)
q4 = sdd.quality_report(mesh4, ref4, m4.with_grad(sdd.GRAD_REFERENCE), ctx=ctx)
out["config4_end_to_end"] = {"mc_points": r4.mc_points, "path_steps": r4.path_steps, "t_stoc_s": r4.t_stoc,
                             "t_sub_s": r4.t_sub, "t_solve_sdd_wall_s": t_sdd, "t_laplacian_s": t_smooth,
                             "t_single_domain_513_s": t_1, "q_max": q4.q_max, "q_mean": q4.q_mean,
                             "r_max": q4.r_max, "r_mean": q4.r_mean, "l_inf": q4.l_inf}

# ---- K3 subdomain solver batches
def solver_batch(g, subs_n, tol, method, n_jobs=None):
    m = sdd.MonitorFunction.shock()
    spec = sdd.GridSpec(UNIT, g, g)
    w = None
    lay = sdd.build_layout(spec, subs_n, subs_n)
    bxy = lay.block_x + 1
    rng = np.random.default_rng(3)
    jobs, bcs = [], []
    n_jobs = n_jobs or 2 * lay.subdomain_count()
    for s in range(n_jobs):
        q = s % lay.subdomain_count()
        i0, j0, nx, ny = lay.subdomain(q % subs_n, q // subs_n)
        v = np.sort(rng.random(4))
        e = lambda a, b: np.linspace(a, b, bxy)
        bcs.append(sdd.EdgeData(e(v[0], v[1]), e(v[2], v[3]), e(v[0], v[2]), e(v[1], v[3])))
        jobs.append((i0, j0, nx, ny))
    w = 1.0 / np.array([[1.0 / (1.0 + 20.0 / np.cosh(50 * (y - 0.5 - 0.15 * np.sin(2 * np.pi * x)))**2)
                         for x in np.linspace(0, 1, g)] for y in np.linspace(0, 1, g)]).ravel()
    res = sdd.solve_dirichlet_batch(w, g, g, 1 / (g - 1), 1 / (g - 1), jobs, bcs,
                                    sdd.SolverConfig(tol=tol, method=method), ctx=ctx)
    st = ctx.last_stats()
    its = np.array([r.iterations for r in res])
    upd = float(np.sum(its) * (bxy - 2) ** 2)
    sec = st["kernel_ms"] / 1e3
    return {"jobs": n_jobs, "n": bxy, "method": method, "tol": tol, "kernel_ms": st["kernel_ms"],
            "iters_mean": float(its.mean()), "iters_max": int(its.max()),
            "point_updates_per_s": upd / sec, "effective_GBps_at_40B": upd * 40 / sec / 1e9,
            "converged": all(r.converged for r in res)}

out["solver_config2_jacobi"] = solver_batch(129, 4, 1e-10, "jacobi")
out["solver_config2_rbsor"] = solver_batch(129, 4, 1e-10, "rbsor")
out["solver_config3_rbsor"] = solver_batch(1025, 8, 1e-10, "rbsor")
out["solver_config3_jacobi"] = solver_batch(1025, 8, 1e-10, "jacobi", n_jobs=16)
out["solver_large_batch_rbsor"] = solver_batch(1025, 8, 1e-10, "rbsor", n_jobs=2048)
print(json.dumps(out, indent=1))

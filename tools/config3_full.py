"""BASELINE config 3 end to end on one B200, at full size: 1025^2 grid, 8x8
subdomains, shock density (analytic drift), all 14,273 interface nodes x 1e6
paths, Euler-Maruyama dt 1e-5 in fp32 with fp64 sums, RB-SOR subdomain solves
to 1e-10, then inversion and mesh quality against the single-domain solve.
Prints one JSON object (profiles/r01_config3_full.json)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

paths = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
m = sdd.MonitorFunction.shock(analytic=True)
spec = sdd.GridSpec(UNIT, 1025, 1025)
lay = sdd.build_layout(spec, 8, 8)
plan = sdd.plan_interface_points("all", 0, m, lay)
cfg = sdd.WalkConfig(scheme="linear", dt=1e-5, walks=paths, seed=1, precision="fp32")
scfg = sdd.SolverConfig(tol=1e-10, method="rbsor")
t0 = time.perf_counter()
r = sdd.solve_sdd(m, lay, plan, cfg, scfg, ctx=ctx)
wall = time.perf_counter() - t0
t1 = time.perf_counter()
lay1 = sdd.build_layout(spec, 1, 1)
single = sdd.solve_sdd(m, lay1, sdd.plan_interface_points("all", 0, m, lay1), sdd.WalkConfig(walks=1), scfg,
                       ctx=ctx)
t_1 = time.perf_counter() - t1
mesh = sdd.invert_mesh(r.xi, r.eta, spec, 1025, 1025, ctx=ctx)
ref = sdd.invert_mesh(single.xi, single.eta, spec, 1025, 1025, ctx=ctx)
q = sdd.quality_report(mesh, ref, m.with_grad(sdd.GRAD_REFERENCE), ctx=ctx)
print(json.dumps({"workload": "BASELINE config 3, full size (1025^2, 8x8, shock, 14,273 nodes x %d paths, "
                  "dt 1e-5 fp32 walks / fp64 sums, RB-SOR 1e-10)" % paths,
                  "t_stoc_s": r.t_stoc, "t_sub_s": r.t_sub, "t_total_s": r.t_stoc + r.t_sub + r.t_smooth,
                  "wall_s": wall, "mc_points": r.mc_points, "path_steps": r.path_steps,
                  "path_steps_per_s": r.path_steps / r.t_stoc, "restarts": r.restarts, "warnings": r.warnings,
                  "subdomain_solves": r.subdomain_solves, "t_single_domain_s": t_1,
                  "q_max": q.q_max, "q_mean": q.q_mean, "r_max": q.r_max, "r_mean": q.r_mean,
                  "l_inf": q.l_inf}, indent=1))

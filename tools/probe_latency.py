"""Per-step latency of the walk kernel when the SM is nearly empty (the
batch tail) against its loaded rate: dumps of n walks at config 1's centre
node (ring, analytic fp64, dt 1e-4) for n = 1, 32, 1024, 16384; the slowest
walk's steps over the kernel time is the per-step latency of one dependent
step chain under that load.  Also the config-1 walk phase's time split."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
out = {}
for analytic in (True, False):
    m = sdd.MonitorFunction.ring(analytic=analytic)
    bd = sdd.make_boundary_data(m, sdd.GridSpec(UNIT, 65, 65))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1, seed=1)
    for n in (1, 32, 1024, 16384):
        best = None
        for _ in range(2):
            d = sdd.walk_dump((0.5, 0.5), 2112, m, UNIT, bd, cfg, 0, n, ctx=ctx)
            st = ctx.last_stats()
            if best is None or st["kernel_ms"] < best[0]:
                best = (st["kernel_ms"], int(d["steps"].max()), int(d["steps"].sum()))
        ms, smax, ssum = best
        out[f"{'analytic' if analytic else 'reference'}_n{n}"] = {
            "kernel_ms": ms, "max_steps": smax, "total_steps": ssum,
            "ns_per_step_of_longest": ms * 1e6 / smax}
        print(json.dumps({f"{'analytic' if analytic else 'reference'}_n{n}": out[f"{'analytic' if analytic else 'reference'}_n{n}"]}), flush=True)
# config 1 walk phase
m = sdd.MonitorFunction.ring(analytic=True)
lay = sdd.build_layout(sdd.GridSpec(UNIT, 65, 65), 2, 2)
px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("equispaced", 31, m, lay))
bd = sdd.make_boundary_data(m, lay.global_)
for walks in (10_000, 40_000):
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=walks, seed=1)
    best = 1e18
    for _ in range(3):
        e = sdd.mc_estimate_batch(np.stack([px, py], 1), pid, m, UNIT, bd, cfg, ctx=ctx)
        best = min(best, ctx.last_stats()["kernel_ms"])
    steps = int(e["path_steps"].sum())
    out[f"config1_walks{walks}"] = {"kernel_ms": best, "path_steps": steps, "rate": steps / best * 1e3}
    print(json.dumps({f"config1_walks{walks}": out[f"config1_walks{walks}"]}), flush=True)
print(json.dumps(out))

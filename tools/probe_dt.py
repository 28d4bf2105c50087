"""Walk-kernel time vs paths per node (intercept = per-batch fixed cost):
config-1 nodes (dt 1e-4) and config-2 nodes (dt 2e-5), analytic ring fp64."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
m = sdd.MonitorFunction.ring(analytic=True)
for dt, grid, subs, place, k, walk_list in ((1e-4, 65, 2, "equispaced", 31, (2500, 10000, 40000, 160000)),
                                            (2e-5, 129, 4, "all", 0, (2000, 8000, 32000))):
    lay = sdd.build_layout(sdd.GridSpec(UNIT, grid, grid), subs, subs)
    px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points(place, k, m, lay))
    bd = sdd.make_boundary_data(m, lay.global_)
    for walks in walk_list:
        cfg = sdd.WalkConfig(scheme="linear", dt=dt, walks=walks, seed=1)
        best = 1e18
        for _ in range(2):
            sdd.mc_estimate_batch(np.stack([px, py], 1), pid, m, UNIT, bd, cfg, ctx=ctx)
            st = ctx.last_stats()
            best = min(best, st["kernel_ms"])
        print(f"dt={dt} walks={walks}: {best:.2f} ms, {st['path_steps'] / best * 1e3:.3e} path-steps/s", flush=True)

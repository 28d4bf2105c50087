"""Where one GPU's share of config 2 at N=8 loses time: walk-kernel time of
the shard (the cost-model plan's rank 0) at 25k/50k/100k paths per node
(the intercept is the batch tail) and with the node launch order reversed
or by index (SDDG_NODE_ORDER) instead of longest-expected first."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
m = sdd.MonitorFunction.ring(analytic=True)
lay = sdd.build_layout(sdd.GridSpec(UNIT, 129, 129), 4, 4)
px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("all", 0, m, lay))
pts = np.stack([px, py], 1)
sel = sdd.shard_plan(pts, m, UNIT, sdd.WalkConfig(scheme="linear", dt=2e-5, walks=100_000), 8)[0] == 0
bd = sdd.make_boundary_data(m, lay.global_)
out = {}
for order in ("lpt", "reverse", "index"):
    if order == "lpt":
        os.environ.pop("SDDG_NODE_ORDER", None)
    else:
        os.environ["SDDG_NODE_ORDER"] = order
    for walks in ((25_000, 50_000, 100_000) if order == "lpt" else (100_000,)):
        cfg = sdd.WalkConfig(scheme="linear", dt=2e-5, walks=walks, seed=1)
        best = None
        for _ in range(2):
            sdd.mc_estimate_batch(pts[sel], pid[sel], m, UNIT, bd, cfg, ctx=ctx)
            st = ctx.last_stats()
            best = st if best is None or st["kernel_ms"] < best["kernel_ms"] else best
        out[f"{order}_{walks}"] = {"kernel_ms": best["kernel_ms"], "path_steps": best["path_steps"],
                                   "rate": best["path_steps"] / best["kernel_ms"] * 1e3}
        print(order, walks, json.dumps(out[f"{order}_{walks}"]), flush=True)
os.environ.pop("SDDG_NODE_ORDER", None)
print(json.dumps(out))

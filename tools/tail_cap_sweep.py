"""When does a small batch's drain end?  Config 1's walk phase (performance
mode) with the K1 -> K1t handoff threshold SDDG_TAIL_PER_SM = 4 ... 1024:
K1 ends about when the live walks fall to the cap (a check point every 256
steps), so K1's time per cap traces the live-walk count over time; the tail
kernel's time shows what it costs to run that many walks one warp each."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
m = sdd.MonitorFunction.ring(analytic=True)
lay = sdd.build_layout(sdd.GridSpec(UNIT, 65, 65), 2, 2)
px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("equispaced", 31, m, lay))
bd = sdd.make_boundary_data(m, lay.global_)
cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=10_000, seed=1)
pts = np.stack([px, py], 1)
caps = [int(c) for c in sys.argv[1:]] or [4, 16, 64, 256, 1024]
for cap in caps:
    os.environ["SDDG_TAIL_PER_SM"] = str(cap)
    best = None
    for _ in range(3):
        sdd.mc_estimate_batch(pts, pid, m, UNIT, bd, cfg, ctx=ctx)
        st = ctx.last_stats()
        if best is None or st["kernel_ms"] < best["kernel_ms"]:
            best = st
    print(json.dumps({"per_sm": cap, "kernel_ms": best["kernel_ms"], "k1_ms": best["kernel_ms"] - best["tail_ms"],
                      "tail_ms": best["tail_ms"], "handoffs": best["tail_handoffs"]}), flush=True)

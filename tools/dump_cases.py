"""Per-path dumps and estimates of the reference-mode (parity) kernels for a
fixed set of cases, saved to an .npz: run once per library build
(SDDG_LIB_PATH) and compare the files bit for bit to show that a change left
the parity mode's arithmetic untouched.  python tools/dump_cases.py OUT.npz"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
out = {}
cases = [("running", sdd.MonitorFunction.running_example(), UNIT),
         ("huang", sdd.MonitorFunction.huang_sloan(), UNIT),
         ("mackenzie", sdd.MonitorFunction.mackenzie(), UNIT),
         ("five", sdd.MonitorFunction.five_ring(), sdd.RectDomain(-1, 1, -1, 1)),
         ("ring_fd", sdd.MonitorFunction.ring(), UNIT),
         ("shock_fd", sdd.MonitorFunction.shock(), UNIT),
         ("twobump_fd", sdd.MonitorFunction.two_bump(), UNIT)]
for name, m, dom in cases:
    bd = sdd.make_boundary_data(m, sdd.GridSpec(dom, 33, 33))
    p = (0.5 * (dom.xmin + dom.xmax) + 0.1, 0.5 * (dom.ymin + dom.ymax) - 0.05)
    for scheme in ("linear", "exponential"):
        cfg = sdd.WalkConfig(scheme=scheme, dt=1e-4, lambda_=1000.0, walks=1, seed=3)
        out[f"{name}_{scheme}"] = sdd.walk_dump(p, 777, m, dom, bd, cfg, 0, 2000, ctx=ctx).view(np.uint8)
np.savez(sys.argv[1], **out)
print(len(out), "cases")

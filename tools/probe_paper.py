"""Where T_stoc goes in the paper-table workload (bench.py --paper-table):
kernel time vs wall of the interface walk batch."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
m = sdd.MonitorFunction.five_ring()
for n in (37, 157):
    spec = sdd.GridSpec(m.domain, n, n)
    lay = sdd.build_layout(spec, 4, 4)
    plan = sdd.plan_interface_points("optimal", 0, m, lay)
    px, py, pid = sdd.interface_nodes(m, lay, plan)
    pts = np.stack([px, py], 1)
    bd = sdd.make_boundary_data(m, spec)
    for walks in (5000, 50000):
        cfg = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=walks, seed=1)
        for rep in range(3):
            t0 = time.perf_counter()
            sdd.mc_estimate_batch(pts, pid, m, m.domain, bd, cfg, ctx=ctx)
            wall = time.perf_counter() - t0
            st = ctx.last_stats()
        print(f"n={n} nodes={len(px)} walks={walks}: wall {wall*1e3:.2f} ms, kernel {st['kernel_ms']:.2f} ms, "
              f"steps {st['path_steps']:.3e} ({st['path_steps']/st['kernel_ms']*1e3:.3e}/s), "
              f"steps/walk {st['path_steps']/len(px)/walks:.0f}")
    for scheme in ("linear",):
        cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=5000, seed=1)
        sdd.mc_estimate_batch(pts, pid, m, m.domain, bd, cfg, ctx=ctx)
        st = ctx.last_stats()
        print(f"  linear dt 1e-4: kernel {st['kernel_ms']:.2f} ms, {st['path_steps']/st['kernel_ms']*1e3:.3e}/s")

"""Throughput of the linear and exponential schemes (performance and reference drift) on the config-2 nodes."""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1310_3435_b200 import sdd
ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
lay = sdd.build_layout(sdd.GridSpec(UNIT, 129, 129), 4, 4)
for name, m in (("ring_an", sdd.MonitorFunction.ring(True)), ("ring_fd", sdd.MonitorFunction.ring(False))):
    px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("all", 0, m, lay))
    bd = sdd.make_boundary_data(m, lay.global_)
    for scheme, lam, walks in (("exponential", 1000.0, 20000), ("exponential", 10000.0, 4000), ("linear", 0, 4000)):
        for prec in (("fp64", "fp32") if name == "ring_an" else ("fp64",)):
            cfg = sdd.WalkConfig(scheme=scheme, dt=2e-5, lambda_=lam or 1000.0, walks=walks, seed=1, precision=prec)
            best = 1e18
            for _ in range(2):
                sdd.mc_estimate_batch(np.stack([px, py], 1), pid, m, UNIT, bd, cfg, ctx=ctx)
                st = ctx.last_stats(); best = min(best, st["kernel_ms"])
            print(f"{name} {scheme} lam={lam} {prec} walks={walks}: {best:.1f} ms {st['path_steps']/best*1e3:.3e} path-steps/s, steps/walk {st['path_steps']/len(px)/walks:.0f}", flush=True)

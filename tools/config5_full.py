"""BASELINE config 5 at its largest size on one B200: 4,096 uniform start
points (numpy seed 1), ring density (analytic drift), dt 1e-5, 1e6 paths per
point in fp32 (4.1e9 paths), plus 1e5 paths per point in fp64.  Prints one
JSON object (profiles/r01_config5_full.json)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
pts = np.clip(np.random.default_rng(1).uniform(0.0, 1.0, size=(4096, 2)), 1e-9, 1 - 1e-9)
pid = np.arange(4096, dtype=np.uint64)
bd = sdd.make_boundary_data(sdd.MonitorFunction.ring(), sdd.GridSpec(UNIT, 129, 129), sdd.BC_IDENTITY)
m = sdd.MonitorFunction.ring(analytic=True)
out = {"workload": "BASELINE config 5: 4096 uniform points, ring, dt 1e-5, identity BCs"}
for prec, paths in (("fp32", 1_000_000), ("fp64", 100_000)):
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-5, walks=paths, seed=1, precision=prec)
    t0 = time.perf_counter()
    e = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd, cfg, ctx=ctx)
    wall = time.perf_counter() - t0
    st = ctx.last_stats()
    out[f"{prec}_{paths}"] = {"paths_total": 4096 * paths, "path_steps": st["path_steps"],
                              "kernel_s": st["kernel_ms"] / 1e3, "wall_s": wall,
                              "path_steps_per_s": st["path_steps"] / (st["kernel_ms"] / 1e3),
                              "launches": st["launches"],
                              "xi_mean_abs_err_vs_x": float(np.mean(np.abs(e["xi"] - pts[:, 0]))),
                              "restarts": int(e["restarts"].sum())}
    print(prec, json.dumps(out[f"{prec}_{paths}"]), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))

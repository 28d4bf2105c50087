"""A/B of the tail kernel (walk_tail.cuh) on tail-bound walk batches: K1 +
tail kernel vs K1 alone (SDDG_NO_TAIL=1), walk-kernel device time, best of 3.

  config1_analytic   BASELINE config 1 walk phase, performance mode
  config1_reference  the same in the bit-faithful parity mode (FD drift)
  config2_shard8     1/8 of config 2's nodes x 1e5 paths: one GPU's share at N=8
  paper157_reference the paper table's 157^2 workload (five-ring, exponential
                     lambda=1000, N=5000, optimal placement), reference drift
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
FIVE = sdd.RectDomain(-1, 1, -1, 1)


def nodes(m, n, s, place, k, dom=UNIT):
    lay = sdd.build_layout(sdd.GridSpec(dom, n, n), s, s)
    px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points(place, k, m, lay))
    return lay, np.stack([px, py], 1), pid


def cases():
    ring_a, ring_r = sdd.MonitorFunction.ring(analytic=True), sdd.MonitorFunction.ring()
    lay1, p1, i1 = nodes(ring_a, 65, 2, "equispaced", 31)
    bd1 = sdd.make_boundary_data(ring_a, lay1.global_)
    c1 = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=10_000, seed=1)
    yield "config1_analytic", ring_a, p1, i1, bd1, c1, UNIT
    yield "config1_reference", ring_r, p1, i1, bd1, c1, UNIT
    lay2, p2, i2 = nodes(ring_a, 129, 4, "all", 0)
    bd2 = sdd.make_boundary_data(ring_a, lay2.global_)
    sel = sdd.shard_plan(p2, ring_a, UNIT, sdd.WalkConfig(scheme="linear", dt=2e-5, walks=100_000), 8)[0] == 0
    yield "config2_shard8", ring_a, p2[sel], i2[sel], bd2, sdd.WalkConfig(scheme="linear", dt=2e-5,
                                                                         walks=100_000, seed=1), UNIT
    five = sdd.MonitorFunction.five_ring()
    lay5, p5, i5 = nodes(five, 157, 4, "optimal", 0, FIVE)
    bd5 = sdd.make_boundary_data(five, lay5.global_)
    yield "paper157_reference", five, p5, i5, bd5, sdd.WalkConfig(scheme="exponential", lambda_=1000.0,
                                                                  walks=5000, seed=1), FIVE


out = {}
only = set(sys.argv[1:])
for name, m, pts, pid, bd, cfg, dom in cases():
    if only and name not in only:
        continue
    res = {}
    for mode in ("tail", "k1_only"):
        if mode == "k1_only":
            os.environ["SDDG_NO_TAIL"] = "1"
        else:
            os.environ.pop("SDDG_NO_TAIL", None)
        best = None
        for _ in range(3):
            e = sdd.mc_estimate_batch(pts, pid, m, dom, bd, cfg, ctx=ctx)
            st = ctx.last_stats()
            if best is None or st["kernel_ms"] < best["kernel_ms"]:
                best = st
        res[mode] = {"kernel_ms": best["kernel_ms"], "path_steps": best["path_steps"],
                     "rate": best["path_steps"] / best["kernel_ms"] * 1e3,
                     "tail_handoffs": best["tail_handoffs"], "tail_ms": best["tail_ms"]}
    os.environ.pop("SDDG_NO_TAIL", None)
    res["speedup"] = res["k1_only"]["kernel_ms"] / res["tail"]["kernel_ms"]
    out[name] = res
    print(name, json.dumps(res), flush=True)
print(json.dumps(out))

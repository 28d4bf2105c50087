"""Run one walk batch of a BASELINE config (for ncu captures):
python tools/walk_once.py {config2|config2fd|config3|config5|five|fivelin|fiveref} {fp64|fp32} WALKS
(five: the paper-table workload's walks -- five-ring density on [-1,1]^2, 77^2
grid split 4x4, exponential stepping lambda = 1000; fivelin: the same nodes
with the linear scheme, dt = 1e-4)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

cfgname, prec, walks = sys.argv[1], sys.argv[2], int(sys.argv[3])
ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
scheme, lam = "linear", 1000.0
if cfgname in ("five", "fivelin", "fiveref"):  # fiveref: the reference-mode drift (parity mode)
    UNIT = sdd.RectDomain(-1, 1, -1, 1)
    m, grid, subs, dt = sdd.MonitorFunction.five_ring(analytic=cfgname != "fiveref"), 77, 4, 1e-4
    scheme = "linear" if cfgname == "fivelin" else "exponential"
elif cfgname == "config3fd":  # shock, the reference's FD drift
    m, grid, subs, dt = sdd.MonitorFunction.shock(analytic=False), 1025, 8, 1e-5
elif cfgname == "running":  # the reference README's running-example density (a builtin drift), exponential
    m, grid, subs, dt = sdd.MonitorFunction.by_name("running"), 129, 4, 2e-5
    scheme, lam = "exponential", 1000.0
elif cfgname == "config3":
    m, grid, subs, dt = sdd.MonitorFunction.shock(analytic=True), 1025, 8, 1e-5
elif cfgname == "config2fd":  # the parity mode: the reference's FD drift of rho = 1/w
    m, grid, subs, dt = sdd.MonitorFunction.ring(analytic=False), 129, 4, 2e-5
elif cfgname == "config2":
    m, grid, subs, dt = sdd.MonitorFunction.ring(analytic=True), 129, 4, 2e-5
else:
    m, grid, subs, dt = sdd.MonitorFunction.ring(analytic=True), 129, 4, 1e-5
spec = sdd.GridSpec(UNIT, grid, grid)
bd = sdd.make_boundary_data(m, spec)
if cfgname == "config5":
    pts = np.clip(np.random.default_rng(1).uniform(0, 1, (4096, 2)), 1e-9, 1 - 1e-9)
    pid = np.arange(4096, dtype=np.uint64)
else:
    lay = sdd.build_layout(spec, subs, subs)
    px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("all", 0, m, lay))
    pts = np.stack([px, py], 1)
scheme = os.environ.get("SDDG_ONCE_SCHEME", scheme)  # e.g. exponential on a linear-scheme workload
cfg = sdd.WalkConfig(scheme=scheme, dt=dt, lambda_=lam, walks=walks, seed=1, precision=prec)
for _ in range(2):
    sdd.mc_estimate_batch(pts, pid, m, UNIT, bd, cfg, ctx=ctx)
    st = ctx.last_stats()
    print(f"{cfgname} {prec} walks={walks}: {st['path_steps'] / (st['kernel_ms'] / 1e3):.4e} path-steps/s")

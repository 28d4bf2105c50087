"""Estimates of performance-mode (analytic drift) walks on a few nodes of the
three BASELINE densities, as bytes (for bit-for-bit comparisons of library
variants, SDDG_LIB_PATH): python tools/dump_est.py OUT"""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1310_3435_b200 import sdd
ctx = sdd.Context(0)
U = sdd.RectDomain(0, 1, 0, 1)
out = []
for m, dt in ((sdd.MonitorFunction.ring(analytic=True), 1e-4), (sdd.MonitorFunction.shock(analytic=True), 2e-5),
              (sdd.MonitorFunction.by_name("two-bump").with_grad(sdd.GRAD_ANALYTIC), 1e-4)):
    bd = sdd.make_boundary_data(m, sdd.GridSpec(U, 65, 65))
    pts = [(0.5, j / 64) for j in range(2, 63, 4)] + [(i / 64, 0.5) for i in range(2, 63, 4)] + [(0.02, 0.03), (0.98, 0.97), (0.5, 0.01)]
    e = sdd.mc_estimate_batch(pts, list(range(len(pts))), m, U, bd, sdd.WalkConfig(scheme="linear", dt=dt, walks=3000, seed=5), ctx=ctx)
    out.append(e.tobytes())
open(sys.argv[1], 'wb').write(b"".join(out))
print("dumped", len(b"".join(out)))

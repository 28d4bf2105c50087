"""Estimates of reference-mode (parity) walks on a few nodes, as bytes (for
bit-for-bit comparisons of library variants): python tools/dump_est_ref.py OUT"""
import sys
sys.path.insert(0, '.')
from paper_1310_3435_b200 import sdd
ctx = sdd.Context(0)
U = sdd.RectDomain(0, 1, 0, 1)
out = []
for m, dt in ((sdd.MonitorFunction.ring(), 1e-4), (sdd.MonitorFunction.shock(), 2e-5),
              (sdd.MonitorFunction.running_example(), 1e-4), (sdd.MonitorFunction.by_name("mackenzie"), 1e-4)):
    bd = sdd.make_boundary_data(m, sdd.GridSpec(U, 65, 65))
    pts = [(0.5, j / 64) for j in range(2, 63, 6)] + [(i / 64, 0.5) for i in range(2, 63, 6)] + [(0.02, 0.03), (0.98, 0.97), (0.5, 0.01)]
    e = sdd.mc_estimate_batch(pts, list(range(len(pts))), m, U, bd, sdd.WalkConfig(scheme="linear", dt=dt, walks=1500, seed=5), ctx=ctx)
    out.append(e.tobytes())
open(sys.argv[1], 'wb').write(b"".join(out))
print("dumped", len(b"".join(out)))

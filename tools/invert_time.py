"""K4 (mesh inversion) kernel time on forward solutions of 513^2 and 1025^2
nodes: the Winslow meshes of the BASELINE densities (the deterministic
single-domain solve; symmetric densities put a few targets per row on a mesh
line, which the fix-up pass handles), an analytic mesh without symmetry (the
parallel passes alone), and the identity mesh (every target on a vertex: the
sequential fix-up does all rows, the worst case).
SDDG_LIB_PATH selects a library variant (tools/ab_walk.sh style)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)
def winslow(m, n):
    """The deterministic single-domain mesh of density m on the n x n grid (RB-SOR)."""
    spec = sdd.GridSpec(UNIT, n, n)
    lay = sdd.build_layout(spec, 1, 1)
    r = sdd.solve_sdd(m, lay, sdd.plan_interface_points("all", 0, m, lay), sdd.WalkConfig(walks=1),
                      sdd.SolverConfig(tol=1e-10, method="rbsor"), ctx=ctx)
    return np.asarray(r.xi).reshape(n, n), np.asarray(r.eta).reshape(n, n)


for n in (513, 1025):
    x, y = np.meshgrid(np.linspace(0, 1, n), np.linspace(0, 1, n))
    cases = {
        "ring (Winslow mesh)": winslow(sdd.MonitorFunction.ring(), n),
        "shock (Winslow mesh)": winslow(sdd.MonitorFunction.shock(), n),
        "two-bump (Winslow mesh)": winslow(sdd.MonitorFunction.by_name("two-bump"), n),
        "analytic, no symmetry": (x + 0.08 * np.sin(2 * np.pi * x) * (1 + 0.5 * np.sin(np.pi * y)) + 0.01 * np.sin(np.pi * x) * y,
                                  y + 0.05 * np.sin(2 * np.pi * y) * (1 + 0.3 * x)),
        "identity (every target on a vertex)": (x, y),
    }
    for name, (xi, eta) in cases.items():
        spec = sdd.GridSpec(UNIT, n, n)
        best = 1e9
        for _ in range(3):
            mesh = sdd.invert_mesh(xi.ravel(), eta.ravel(), spec, n, n, ctx=ctx)
            st = ctx.last_stats()
            best = min(best, st["kernel_ms"])
        print(f"{n}^2 {name}: K4 {best:.3f} ms, fix-up rows {st['tail_handoffs']}, targets located again "
              f"{st['path_steps']}, checksum {float(np.sum(mesh.x) + np.sum(mesh.y)):.12f}", flush=True)

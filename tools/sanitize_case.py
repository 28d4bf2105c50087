"""Small end-to-end case for compute-sanitizer runs (one tool per gpurun call):
walk dump + estimates (K1/K2), the tail kernel (K1t), solve_sdd (K3), large
solver (K3b), inversion + quality (K4/K5), smoothing (K6/K7), a tabulated
density, the literal SDE form, and the multi-GPU contexts (pack/scatter
kernels, a one-rank NCCL all-gather, device-copy exchange)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
U = sdd.RectDomain(0, 1, 0, 1)
for m in (sdd.MonitorFunction.ring(), sdd.MonitorFunction.ring(analytic=True)):
    spec = sdd.GridSpec(U, 33, 33)
    bd = sdd.make_boundary_data(m, spec)
    sdd.walk_dump((0.5, 0.5), 528, m, U, bd, sdd.WalkConfig(scheme="linear", dt=1e-3, walks=1, seed=1), 0, 64, ctx=ctx)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("equispaced", 5, m, lay)
    r = sdd.solve_sdd(m, lay, plan, sdd.WalkConfig(scheme="linear", dt=1e-3, walks=64, seed=1),
                      sdd.SolverConfig(tol=1e-10, method="rbsor"), ctx=ctx)
    sdd.solve_sdd(m, lay, plan, sdd.WalkConfig(scheme="exponential", lambda_=300, walks=64, seed=1,
                                                precision="fp64"), sdd.SolverConfig(tol=1e-10), ctx=ctx)
mf = sdd.MonitorFunction.ring(analytic=True)
sdd.mc_estimate_batch([(0.3, 0.4), (0.6, 0.7)], [1, 2], mf, U, sdd.make_boundary_data(mf, sdd.GridSpec(U, 17, 17)),
                      sdd.WalkConfig(scheme="linear", dt=1e-3, walks=300, seed=3, precision="fp32"), ctx=ctx)
mesh = sdd.invert_mesh(r.xi, r.eta, spec, 33, 33, ctx=ctx)
sdd.quality_report(mesh, mesh, m, ctx=ctx)
sdd.perona_malik(r.xi, r.eta, spec, sdd.SmoothConfig(k=1000.0, dt=1e-4, steps=3, scope="per_subdomain"), lay, ctx=ctx)
sdd.smooth_interface(np.linspace(0, 1, 33) ** 2, 5, ctx=ctx)
w = np.ones(193 * 193)
x = np.linspace(0, 1, 193)
sdd.solve_dirichlet(w, 193, 193, 1 / 192, 1 / 192, sdd.EdgeData(x, x, np.zeros(193), np.ones(193)),
                    sdd.SolverConfig(tol=1e-8, method="rbsor"), ctx=ctx)
# K1t: 700 walks, all handed over at their 256th step
sdd.walk_dump((0.5, 0.5), 2112, sdd.MonitorFunction.ring(analytic=True), U,
              sdd.make_boundary_data(sdd.MonitorFunction.ring(), sdd.GridSpec(U, 65, 65)),
              sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1, seed=1), 0, 700, ctx=ctx)
sdd.walk_dump((0.5, 0.5), 2112, sdd.MonitorFunction.ring(), U,
              sdd.make_boundary_data(sdd.MonitorFunction.ring(), sdd.GridSpec(U, 65, 65)),
              sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1, seed=1), 0, 300, ctx=ctx)
# tabulated density (reference FD and analytic) and the literal form
xx = np.linspace(0, 1, 17)
XX, YY = np.meshgrid(xx, xx)
mt = sdd.MonitorFunction.tabulated(1.0 + XX * YY, U)
bdt = sdd.make_boundary_data(mt, sdd.GridSpec(U, 17, 17))
sdd.mc_estimate_batch([(0.3, 0.4)], [5], mt, U, bdt, sdd.WalkConfig(scheme="linear", dt=1e-3, walks=256, seed=1),
                      ctx=ctx)
sdd.mc_estimate_batch([(0.3, 0.4)], [5], mt.with_grad(sdd.GRAD_ANALYTIC), U, bdt,
                      sdd.WalkConfig(scheme="exponential", walks=256, seed=1), ctx=ctx)
sdd.mc_estimate_batch([(0.3, 0.4)], [5], mf, U, bdt,
                      sdd.WalkConfig(scheme="linear", dt=1e-3, walks=256, seed=1, form="literal"), ctx=ctx)
# multi-GPU contexts on this one device
for team in (sdd.Context.multi([0, 0]), sdd.Context.dist(0, 0, 1, sdd.nccl_unique_id())):
    lay4 = sdd.build_layout(sdd.GridSpec(U, 33, 33), 4, 2)
    sdd.solve_sdd(mf, lay4, sdd.plan_interface_points("equispaced", 7, mf, lay4),
                  sdd.WalkConfig(scheme="linear", dt=1e-3, walks=128, seed=1),
                  sdd.SolverConfig(tol=1e-10, method="rbsor"), ctx=team)
    team.close()
print("sanitize case done")

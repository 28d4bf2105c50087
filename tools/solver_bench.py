"""K3 batches of the BASELINE subdomain solves (shock weights), fixed vs
adaptive SOR factor: python tools/solver_bench.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)
UNIT = sdd.RectDomain(0, 1, 0, 1)


def batch(g, subs_n, n_jobs=None, omega=0.0, tol=1e-10):
    spec = sdd.GridSpec(UNIT, g, g)
    lay = sdd.build_layout(spec, subs_n, subs_n)
    bxy = lay.block_x + 1
    rng = np.random.default_rng(3)
    jobs, bcs = [], []
    n_jobs = n_jobs or 2 * lay.subdomain_count()
    for s in range(n_jobs):
        q = s % lay.subdomain_count()
        jobs.append(lay.subdomain(q % subs_n, q // subs_n))
        v = np.sort(rng.random(4))
        e = lambda a, b: np.linspace(a, b, bxy)  # noqa: E731
        bcs.append(sdd.EdgeData(e(v[0], v[1]), e(v[2], v[3]), e(v[0], v[2]), e(v[1], v[3])))
    x = np.linspace(0, 1, g)
    X, Y = np.meshgrid(x, x)
    w = (1.0 + 20.0 / np.cosh(50 * (Y - 0.5 - 0.15 * np.sin(2 * np.pi * X))) ** 2).ravel()
    cfg = sdd.SolverConfig(tol=tol, method="rbsor", omega=omega)
    for _ in range(2):
        res = sdd.solve_dirichlet_batch(w, g, g, 1 / (g - 1), 1 / (g - 1), jobs, bcs, cfg, ctx=ctx)
        st = ctx.last_stats()
    its = np.array([r.iterations for r in res])
    upd = float(np.sum(its) * (bxy - 2) ** 2)
    sec = st["kernel_ms"] / 1e3
    return {"jobs": n_jobs, "n": bxy, "omega": "adaptive" if omega <= 0 else omega,
            "kernel_ms": st["kernel_ms"], "iters_mean": float(its.mean()), "iters_max": int(its.max()),
            "effective_GBps_at_40B": upd * 40 / sec / 1e9, "converged": all(r.converged for r in res),
            "fields": [r.values for r in res[:2]]}


out = {}
for name, (g, s, nj) in {"config2": (129, 4, None), "config3": (1025, 8, None),
                         "large_2048": (1025, 8, 2048)}.items():
    h = 1.0 / (g // s)
    w_lap = 2.0 / (1.0 + np.sin(np.pi * h))
    a, f = batch(g, s, nj, 0.0), batch(g, s, nj, w_lap)
    diff = max(float(np.max(np.abs(x - y))) for x, y in zip(a.pop("fields"), f.pop("fields")))
    out[name] = {"adaptive": a, "fixed": f, "max_field_diff": diff}
print(json.dumps(out, indent=1))

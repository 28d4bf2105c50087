"""A/B of the RB-SOR factor: the per-job Rayleigh-quotient estimate (omega = 0,
the default) against the constant-coefficient grid formula (omega < 0), on the
solver batches of bench.py (config-3 shock weights, 128 and 2048 x 129^2), the
config-4 two-bump blocks (16 x 2 x 129^2) and config 4's single-domain 513^2
solve (K3b).  Prints ms, sweeps (mean/max) and the largest field difference.
python tools/omega_ab.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_3435_b200 import sdd  # noqa: E402

ctx = sdd.Context(0)


def weights(kind, g):
    x = np.linspace(0, 1, g)
    X, Y = np.meshgrid(x, x)
    if kind == "shock":
        return (1.0 + 20.0 / np.cosh(50 * (Y - 0.5 - 0.15 * np.sin(2 * np.pi * X))) ** 2).ravel()
    return (1 + 15 * np.exp(-100 * ((X - .3) ** 2 + (Y - .3) ** 2))
            + 15 * np.exp(-100 * ((X - .7) ** 2 + (Y - .6) ** 2))).ravel()


def batch(kind, g, subs_n, n_jobs):
    spec = sdd.GridSpec(sdd.RectDomain(0, 1, 0, 1), g, g)
    lay = sdd.build_layout(spec, subs_n, subs_n)
    bxy = lay.block_x + 1
    rng = np.random.default_rng(3)
    jobs, bcs = [], []
    for s in range(n_jobs):
        q = s % lay.subdomain_count()
        jobs.append(lay.subdomain(q % subs_n, q // subs_n))
        v = np.sort(rng.random(4))
        e = lambda a, b: np.linspace(a, b, bxy)  # noqa: E731
        bcs.append(sdd.EdgeData(e(v[0], v[1]), e(v[2], v[3]), e(v[0], v[2]), e(v[1], v[3])))
    return jobs, bcs


out = {}
cases = [("config3_batch", "shock", 1025, 8, 128), ("batch_2048", "shock", 1025, 8, 2048),
         ("config4_blocks", "bump", 513, 4, 32), ("config4_single", "bump", 513, 1, 2)]
for name, kind, g, subs_n, n_jobs in cases:
    w = weights(kind, g)
    jobs, bcs = batch(kind, g, subs_n, n_jobs)
    row = {}
    fields = {}
    for label, om in (("grid_formula", -1.0), ("per_job", 0.0)):
        cfg = sdd.SolverConfig(tol=1e-10, method="rbsor", omega=om)
        best = None
        for _ in range(3):
            res = sdd.solve_dirichlet_batch(w, g, g, 1 / (g - 1), 1 / (g - 1), jobs, bcs, cfg, ctx=ctx)
            ms = ctx.last_stats()["kernel_ms"]
            best = ms if best is None else min(best, ms)
        its = np.array([r.iterations for r in res])
        fields[label] = np.concatenate([np.asarray(r.values).ravel()
                                        for r in res])
        row[label] = {"ms": round(best, 3), "sweeps_mean": float(its.mean()), "sweeps_max": int(its.max()),
                      "converged": bool(all(r.converged for r in res))}
    row["max_abs_diff"] = float(np.max(np.abs(fields["grid_formula"] - fields["per_job"])))
    row["speedup"] = row["grid_formula"]["ms"] / row["per_job"]["ms"]
    out[name] = row
    print(name, json.dumps(row), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/omega_ab.json", "w") as f:
    json.dump(out, f, indent=1)

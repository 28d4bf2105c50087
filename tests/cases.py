"""Shared test cases: the golden-fixture definitions of tests/golden/make_golden.py
re-exported for the tests, plus converters between the oracle and product APIs."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from golden.make_golden import DENSITIES, DUMPS, ESTIMATES  # noqa: E402,F401

from oracle import bindings as B  # noqa: E402


def tables_from_flat(flat, nx, ny, dom):
    o = np.cumsum([0, nx, nx, ny, ny, nx, nx, ny, ny])
    parts = [flat[o[k]:o[k + 1]] for k in range(8)]
    return B.Tables(dom, nx, ny, parts[:4], parts[4:])


def sdd_monitor(kind, analytic=False):
    from paper_1310_3435_b200 import sdd
    return {B.CONSTANT: sdd.MonitorFunction.constant(), B.RUNNING: sdd.MonitorFunction.running_example(),
            B.HUANG_SLOAN: sdd.MonitorFunction.huang_sloan(), B.MACKENZIE: sdd.MonitorFunction.mackenzie(),
            B.FIVE_RING: sdd.MonitorFunction.five_ring()}.get(kind) or sdd.MonitorFunction.weight(kind, analytic)


def sdd_boundary(tables):
    from paper_1310_3435_b200 import sdd
    d = tables.dom
    spec = sdd.GridSpec(sdd.RectDomain(d.xmin, d.xmax, d.ymin, d.ymax), tables.nx, tables.ny)
    return sdd.BoundaryData(spec, sdd.EdgeData(*tables.f), sdd.EdgeData(*tables.g))


def sdd_walk_cfg(kw, walks=1):
    from paper_1310_3435_b200 import sdd
    return sdd.WalkConfig(scheme="exponential" if kw.get("scheme") == "exp" else "linear",
                          dt=kw.get("dt", 1e-4), lambda_=kw.get("lam", 1000.0),
                          walks=kw.get("walks", walks), seed=kw.get("seed", 1),
                          max_steps=kw.get("max_steps", 10_000_000),
                          bridge_test=kw.get("bridge", True))


def plan_from_flat(flat):
    lines, k = [], 0
    while k < len(flat):
        v, fi, n = int(flat[k]), int(flat[k + 1]), int(flat[k + 2])
        lines.append((bool(v), fi, [int(x) for x in flat[k + 3:k + 3 + n]]))
        k += 3 + n
    return lines

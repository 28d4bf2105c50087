"""Pin the CPU oracle (oracle/sdd_oracle.c) to the reference's own outputs.

Every array in tests/golden/golden.npz was produced by the unmodified
reference library (tests/golden/make_golden.py); the C restatement must
reproduce each one bit for bit.  Where oracle/_ref is built, the reference is
re-run too, which checks that the fixtures are current.
"""
import numpy as np
import pytest

from cases import DENSITIES, DUMPS, ESTIMATES, plan_from_flat, tables_from_flat
from oracle import bindings as B

UNIT = B.Domain(0, 1, 0, 1)
FIVE = B.Domain(-1, 1, -1, 1)


def test_philox_blocks(golden, oracle):
    for row, want in zip(golden["philox_in"], golden["philox_out"]):
        got = oracle.philox_block(int(row[0]), int(row[1]), [int(v) for v in row[2:]])
        assert got == [int(v) for v in want]


def test_streams_u64_and_normals(golden, oracle):
    for k, s in enumerate(golden["stream_keys"]):
        key = [int(v) for v in s]
        assert np.array_equal(oracle.stream_u64(*key, 64), golden["stream_u64"][k])
        assert np.array_equal(oracle.stream_normals(*key, 32), golden["stream_normals"][k])


def test_stream_keying_property(oracle):
    # proj/tests/test_sde.cpp:41-55: reproducible, and keyed by walk/seed/point
    a = oracle.stream_u64(1, 7, 3, 0, 16)
    assert np.array_equal(a, oracle.stream_u64(1, 7, 3, 0, 16))
    for other in [(1, 7, 4, 0), (2, 7, 3, 0), (1, 8, 3, 0), (1, 7, 3, 1)]:
        assert not np.array_equal(a, oracle.stream_u64(*other, 16))


@pytest.mark.parametrize("name,kind,dom", DENSITIES, ids=[d[0] for d in DENSITIES])
def test_density_and_drift(golden, oracle, name, kind, dom):
    x, y = golden[f"dens_{name}_xy"]
    rho, bx, by = oracle.rho_drift(B.density(kind), x, y)
    want = golden[f"dens_{name}_out"]
    assert np.array_equal(rho, want[0])
    assert np.array_equal(bx, want[1])
    assert np.array_equal(by, want[2])


@pytest.mark.parametrize("key", ["ring_65", "shock_129", "twobump_33", "running_29", "five_ring_17", "five_ring_33",
                                 "constant_33", "huang_sloan_33", "mackenzie_33", "running17_17"])
def test_boundary_tables(golden, oracle, key):
    name, n = key.rsplit("_", 1)
    n = int(n)
    kind = dict((d[0], d[1]) for d in DENSITIES)["running" if name == "running17" else name]
    dom = FIVE if kind == B.FIVE_RING else UNIT
    t = oracle.make_boundary(B.density(kind), dom, n, n)
    assert np.array_equal(np.concatenate(t.f + t.g), golden[f"tables_{key}"])


@pytest.mark.parametrize("case", DUMPS, ids=[d[0] for d in DUMPS])
def test_walk_dumps(golden, oracle, case):
    name, kind, n, kw, p, pid, nw = case
    dom = FIVE if kind == B.FIVE_RING else UNIT
    t = oracle.make_boundary(B.density(kind), dom, n, n)
    got = oracle.walk_dump(B.density(kind), dom, t, B.walk_cfg(**kw), p[0], p[1], pid, 0, nw)
    want = golden[f"dump_{name}"].view(B.PATH_DTYPE)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    if name == "constant_restart":
        assert (want["epoch"] > 0).any()


@pytest.mark.parametrize("case", ESTIMATES, ids=[e[0] for e in ESTIMATES])
def test_estimates(golden, oracle, case):
    name, kind, n, kw, pts, pids = case
    t = oracle.make_boundary(B.density(kind), UNIT, n, n)
    got = oracle.mc_estimate_batch(B.density(kind), UNIT, t, B.walk_cfg(**kw), [p[0] for p in pts],
                                   [p[1] for p in pts], pids, threads=2)
    want = golden[f"est_{name}"].view(B.EST_DTYPE)
    for f in ("xi", "eta", "se_xi", "se_eta", "walks", "restarts", "warn", "edge_hits"):
        assert np.array_equal(got[f], want[f]), f


def test_estimate_equals_chunked_sum_of_dumps(oracle):
    # mc_estimate = fixed chunk-order sum of run_walk results (sde.cpp:201-229)
    t = oracle.make_boundary(B.density(B.RUNNING), UNIT, 17, 17)
    cfg = B.walk_cfg(scheme="exp", lam=1000.0, seed=9, walks=600)
    d = oracle.walk_dump(B.density(B.RUNNING), UNIT, t, cfg, 0.4, 0.4, 3, 0, 600)
    e = oracle.mc_estimate_batch(B.density(B.RUNNING), UNIT, t, cfg, [0.4], [0.4], [3])[0]
    tot = 0.0
    for c in range(0, 600, 256):
        s = 0.0
        for v in d["f"][c:c + 256]:
            s += v
        tot += s
    assert tot / 600 == e["xi"]


@pytest.mark.parametrize("name", ["ring17_t10", "running33x17_t8", "twobump17_noblend",
                                  "ring33_maxit", "shock33_t13"])
def test_solve_dirichlet(golden, oracle, name):
    meta = {"ring17_t10": (B.RING_W, 17, 17, 1e-10, 0, True),
            "running33x17_t8": (B.RUNNING, 33, 17, 1e-8, 0, True),
            "twobump17_noblend": (B.TWOBUMP_W, 17, 17, 1e-9, 0, False),
            "ring33_maxit": (B.RING_W, 33, 33, 1e-12, 50, True),
            "shock33_t13": (B.SHOCK_W, 33, 33, 1e-13, 0, True)}[name]
    kind, nx, ny, tol, mi, blend = meta
    w = oracle.weight_values(B.density(kind), UNIT, nx, ny)
    assert np.array_equal(w, golden[f"solve_{name}_w"])
    b = [oracle.solve_1d_boundary(B.density(kind), UNIT, nx, ny, e) for e in range(4)]
    fb = {"xi": [b[0], b[1], np.zeros(ny), np.ones(ny)], "eta": [np.zeros(nx), np.ones(nx), b[2], b[3]]}
    for fld in ("xi", "eta"):
        u, it, fu, cv = oracle.solve_dirichlet(w, nx, ny, 1.0 / (nx - 1), 1.0 / (ny - 1), *fb[fld],
                                               tol=tol, max_iters=mi, init_blend=blend)
        assert np.array_equal(u, golden[f"solve_{name}_{fld}_u"])
        info = golden[f"solve_{name}_{fld}_info"]
        assert it == int(info[0]) and fu == info[1] and cv == bool(info[2])


@pytest.mark.parametrize("name,kind,n,sx,st,k", [
    ("running29_all", B.RUNNING, 29, 2, 0, 0), ("running29_eq7", B.RUNNING, 29, 2, 1, 7),
    ("running29_opt", B.RUNNING, 29, 2, 2, 0), ("constant29_opt", B.CONSTANT, 29, 2, 2, 0),
    ("ring65_eq31", B.RING_W, 65, 2, 1, 31), ("twobump513_opt", B.TWOBUMP_W, 513, 4, 2, 0),
    ("five157_opt", B.FIVE_RING, 157, 4, 2, 0), ("shock129_eq40", B.SHOCK_W, 129, 4, 1, 40)])
def test_plans(golden, oracle, name, kind, n, sx, st, k):
    dom = FIVE if kind == B.FIVE_RING else UNIT
    want = plan_from_flat(golden[f"plan_{name}"])
    for vertical, fixed, nodes in want:
        assert oracle.plan_line(st, k, B.density(kind), dom, n, n, vertical, fixed) == nodes


def test_equispaced_golden_indices(oracle):
    # proj/tests/test_decomposition.cpp:76-82
    got = oracle.plan_line(1, 7, B.density(B.RUNNING), UNIT, 29, 29, True, 14)
    assert got == [4, 7, 11, 14, 18, 21, 25]


def test_reference_regenerates_fixtures(golden, refimpl):
    # fixtures are current: the reference reproduces a sample of them now
    for k, s in enumerate(golden["stream_keys"]):
        assert np.array_equal(refimpl.stream_u64(*[int(v) for v in s], 64), golden["stream_u64"][k])
    name, kind, n, kw, p, pid, nw = DUMPS[0]
    t = tables_from_flat(golden["tables_ring_65"], 65, 65, UNIT)
    d = refimpl.walk_dump(B.density(kind), UNIT, t, B.walk_cfg(**kw), p[0], p[1], pid, 0, nw)
    assert np.array_equal(d.view(np.uint8), golden[f"dump_{name}"])

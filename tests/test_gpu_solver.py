"""GPU parity of the batched subdomain solver (K3) through the C-ABI.

Jacobi mode performs the reference iteration (proj/src/detsolver.cpp:150-189)
with the same rounding sequence: fields, iteration counts, final updates and
convergence flags must be bit-identical to the reference's.  Red-black SOR
must land within 1e-10 of the reference's fixed point (BASELINE.json:
"subdomain meshes must match within 1e-10 in fp64").  The dense direct-solve
oracle follows proj/tests/test_detsolver.cpp:35-109.
"""
import numpy as np
import pytest

from oracle import bindings as B
from paper_1310_3435_b200 import sdd

pytestmark = pytest.mark.gpu
UNIT = B.Domain(0, 1, 0, 1)
SOLVES = {"ring17_t10": (B.RING_W, 17, 17, 1e-10, 0, True),
          "running33x17_t8": (B.RUNNING, 33, 17, 1e-8, 0, True),
          "twobump17_noblend": (B.TWOBUMP_W, 17, 17, 1e-9, 0, False),
          "ring33_maxit": (B.RING_W, 33, 33, 1e-12, 50, True),
          "shock33_t13": (B.SHOCK_W, 33, 33, 1e-13, 0, True)}


def _bc(oracle, kind, nx, ny, field):
    b = [oracle.solve_1d_boundary(B.density(kind), UNIT, nx, ny, e) for e in range(4)]
    if field == "xi":
        return sdd.EdgeData(b[0], b[1], np.zeros(ny), np.ones(ny))
    return sdd.EdgeData(np.zeros(nx), np.ones(nx), b[2], b[3])


@pytest.mark.parametrize("name", list(SOLVES))
def test_jacobi_bit_identical_to_reference(golden, oracle, ctx, name):
    kind, nx, ny, tol, mi, blend = SOLVES[name]
    w = golden[f"solve_{name}_w"]
    for fld in ("xi", "eta"):
        r = sdd.solve_dirichlet(w, nx, ny, 1.0 / (nx - 1), 1.0 / (ny - 1), _bc(oracle, kind, nx, ny, fld),
                                sdd.SolverConfig(tol=tol, max_iters=mi, init_blend=blend), ctx=ctx)
        info = golden[f"solve_{name}_{fld}_info"]
        assert np.array_equal(r.values, golden[f"solve_{name}_{fld}_u"])
        assert r.iterations == int(info[0]) and r.final_update == info[1]
        assert r.converged == bool(info[2])
        if not r.converged:
            assert r.warning.startswith("Jacobi reached max_iters=50")


def dense_solve(w, nx, ny, bc):
    """Gaussian elimination over the interior (proj/tests/test_detsolver.cpp:35-109)."""
    hx, hy = 1.0 / (nx - 1), 1.0 / (ny - 1)
    W = w.reshape(ny, nx)
    U = np.zeros((ny, nx))
    U[0, :], U[-1, :], U[:, 0], U[:, -1] = bc.bottom, bc.top, bc.left, bc.right
    m = (nx - 2) * (ny - 2)
    A = np.zeros((m, m))
    rhs = np.zeros(m)
    unk = lambda i, j: (j - 1) * (nx - 2) + (i - 1)
    for j in range(1, ny - 1):
        for i in range(1, nx - 1):
            r = unk(i, j)
            cs = {(i + 1, j): 0.5 * (W[j, i] + W[j, i + 1]) / hx ** 2,
                  (i - 1, j): 0.5 * (W[j, i] + W[j, i - 1]) / hx ** 2,
                  (i, j + 1): 0.5 * (W[j, i] + W[j + 1, i]) / hy ** 2,
                  (i, j - 1): 0.5 * (W[j, i] + W[j - 1, i]) / hy ** 2}
            A[r, r] = sum(cs.values())
            for (ii, jj), c in cs.items():
                if ii in (0, nx - 1) or jj in (0, ny - 1):
                    rhs[r] += c * U[jj, ii]
                else:
                    A[r, unk(ii, jj)] = -c
    U[1:-1, 1:-1] = np.linalg.solve(A, rhs).reshape(ny - 2, nx - 2)
    return U.ravel()


@pytest.mark.parametrize("method", ["jacobi", "rbsor"])
@pytest.mark.parametrize("kind", [B.RING_W, B.RUNNING, B.SHOCK_W])
def test_matches_dense_direct_solve(oracle, ctx, method, kind):
    nx = ny = 17
    w = oracle.weight_values(B.density(kind), UNIT, nx, ny)
    for fld in ("xi", "eta"):
        bc = _bc(oracle, kind, nx, ny, fld)
        r = sdd.solve_dirichlet(w, nx, ny, 1 / 16, 1 / 16, bc, sdd.SolverConfig(tol=1e-13, method=method),
                                ctx=ctx)
        assert np.max(np.abs(r.values - dense_solve(w, nx, ny, bc))) <= 1e-10


@pytest.mark.parametrize("kind,n", [(B.RING_W, 33), (B.SHOCK_W, 33), (B.TWOBUMP_W, 65)])
def test_rbsor_within_1e10_of_reference_jacobi(oracle, ctx, kind, n):
    w = oracle.weight_values(B.density(kind), UNIT, n, n)
    for fld in ("xi", "eta"):
        bc = _bc(oracle, kind, n, n, fld)
        u_ref, *_ = oracle.solve_dirichlet(w, n, n, 1 / (n - 1), 1 / (n - 1), *bc.arrays(), tol=1e-13)
        r = sdd.solve_dirichlet(w, n, n, 1 / (n - 1), 1 / (n - 1), bc,
                                sdd.SolverConfig(tol=1e-13, method="rbsor"), ctx=ctx)
        assert r.converged
        assert np.max(np.abs(r.values - u_ref)) <= 1e-10


def test_linear_data_reproduced_exactly(ctx):
    # proj/tests/test_detsolver.cpp:142-153: uniform weight, affine data
    n = 21
    x = np.arange(n) / (n - 1)
    f = lambda X, Y: 0.3 + 0.5 * X - 0.2 * Y
    bc = sdd.EdgeData(f(x, 0.0), f(x, 1.0), f(0.0, x), f(1.0, x))
    r = sdd.solve_dirichlet(np.ones(n * n), n, n, 1 / (n - 1), 1 / (n - 1), bc,
                            sdd.SolverConfig(tol=1e-14), ctx=ctx)
    X, Y = np.meshgrid(x, x)
    assert np.max(np.abs(r.values - f(X, Y).ravel())) <= 1e-12


def test_maximum_principle_and_transpose_symmetry(oracle, ctx):
    # proj/tests/test_detsolver.cpp:186-202, 246-280
    n = 25
    w = oracle.weight_values(B.density(B.RUNNING), UNIT, n, n)
    bc = _bc(oracle, B.RUNNING, n, n, "xi")
    a = sdd.solve_dirichlet(w, n, n, 1 / 24, 1 / 24, bc, sdd.SolverConfig(tol=1e-10), ctx=ctx)
    assert a.values.min() >= 0.0 and a.values.max() <= 1.0
    wt = w.reshape(n, n).T.ravel()
    bct = sdd.EdgeData(bc.left, bc.right, bc.bottom, bc.top)
    b = sdd.solve_dirichlet(wt, n, n, 1 / 24, 1 / 24, bct, sdd.SolverConfig(tol=1e-10), ctx=ctx)
    assert np.array_equal(a.values.reshape(n, n).T.ravel(), b.values)


def test_init_independence(oracle, ctx):
    # proj/tests/test_detsolver.cpp:219-230
    n = 17
    w = oracle.weight_values(B.density(B.RING_W), UNIT, n, n)
    bc = _bc(oracle, B.RING_W, n, n, "eta")
    a = sdd.solve_dirichlet(w, n, n, 1 / 16, 1 / 16, bc, sdd.SolverConfig(tol=1e-10), ctx=ctx)
    b = sdd.solve_dirichlet(w, n, n, 1 / 16, 1 / 16, bc, sdd.SolverConfig(tol=1e-10, init_blend=False), ctx=ctx)
    assert np.max(np.abs(a.values - b.values)) <= 10 * 1e-10


def test_errors(ctx):
    n = 9
    x = np.arange(n) / (n - 1)
    good = sdd.EdgeData(x, x, np.zeros(n), np.ones(n))
    with pytest.raises(sdd.ValidationError, match="corner"):
        sdd.solve_dirichlet(np.ones(n * n), n, n, 0.125, 0.125, sdd.EdgeData(x, x, np.ones(n), np.ones(n)),
                            sdd.SolverConfig(), ctx=ctx)
    with pytest.raises(sdd.EvaluationError):
        w = np.ones(n * n)
        w[5] = -1.0
        sdd.solve_dirichlet(w, n, n, 0.125, 0.125, good, sdd.SolverConfig(), ctx=ctx)
    with pytest.raises(sdd.ValidationError):
        sdd.solve_dirichlet(np.ones(n * n), n, n, 0.125, 0.125, good, sdd.SolverConfig(tol=0.0), ctx=ctx)
    with pytest.raises(sdd.ValidationError):
        sdd.solve_dirichlet(np.ones(4), 2, 2, 1.0, 1.0, sdd.EdgeData(*[np.zeros(2)] * 4), sdd.SolverConfig(),
                            ctx=ctx)


def test_empty_batch_is_a_no_op(ctx):
    for method in ("jacobi", "rbsor"):
        assert sdd.solve_dirichlet_batch(np.ones(9 * 9), 9, 9, 0.125, 0.125, [], [],
                                         sdd.SolverConfig(method=method), ctx=ctx) == []


def test_config3_batch_rbsor_against_reference_jacobi_sample(oracle, ctx):
    # BASELINE config 3: 64 subdomains x 2 fields of 129^2 in one launch;
    # two of them against the reference iteration at tol 1e-13
    g = 1025
    w = oracle.weight_values(B.density(B.SHOCK_W), UNIT, g, g)
    subs, bcs = [], []
    rng = np.random.default_rng(3)
    for s in range(64):
        a, b = s % 8, s // 8
        for fld in range(2):
            i0, j0 = a * 128, b * 128
            edge = lambda lo, hi: np.linspace(lo, hi, 129)
            v0, v1, v2, v3 = np.sort(rng.random(4))
            bcs.append(sdd.EdgeData(edge(v0, v1), edge(v2, v3), edge(v0, v2), edge(v1, v3)))
            subs.append((i0, j0, 129, 129))
    res = sdd.solve_dirichlet_batch(w, g, g, 1 / 1024, 1 / 1024, subs, bcs,
                                    sdd.SolverConfig(tol=1e-13, method="rbsor"), ctx=ctx)
    assert all(r.converged for r in res)
    for k in (0, 77):
        i0, j0, nx, ny = subs[k]
        wl = w.reshape(g, g)[j0:j0 + ny, i0:i0 + nx].ravel()
        u_ref, *_ = oracle.solve_dirichlet(wl, nx, ny, 1 / 1024, 1 / 1024, *bcs[k].arrays(), tol=1e-13)
        assert np.max(np.abs(res[k].values - u_ref)) <= 1e-10


@pytest.mark.parametrize("nx,ny", [(129, 129), (129, 97), (160, 130)])
def test_cluster_solver_matches_single_cta_solver(oracle, ctx, monkeypatch, nx, ny):
    # K3c (one thread-block cluster per job, strips + DSMEM halos) performs
    # the single-CTA K3's red-black iteration (same weights, same update
    # expression, exact max): identical iterates, bit for bit; shapes cover
    # odd/even row lengths and a short last strip
    g = 257
    w = oracle.weight_values(B.density(B.SHOCK_W), UNIT, g, g)
    rng = np.random.default_rng(nx * ny)
    subs, bcs = [], []
    for k in range(6):
        v0, v1, v2, v3 = np.sort(rng.random(4))
        ex = lambda lo, hi: np.linspace(lo, hi, nx)  # noqa: E731
        ey = lambda lo, hi: np.linspace(lo, hi, ny)  # noqa: E731
        bcs.append(sdd.EdgeData(ex(v0, v1), ex(v2, v3), ey(v0, v2), ey(v1, v3)))
        subs.append(((k * 17) % (g - nx), (k * 29) % (g - ny), nx, ny))
    cfg = sdd.SolverConfig(tol=1e-13, method="rbsor")
    a = sdd.solve_dirichlet_batch(w, g, g, 1 / (g - 1), 1 / (g - 1), subs, bcs, cfg, ctx=ctx)
    monkeypatch.setenv("SDDG_NO_CLUSTER_SOLVER", "1")
    b = sdd.solve_dirichlet_batch(w, g, g, 1 / (g - 1), 1 / (g - 1), subs, bcs, cfg, ctx=ctx)
    for ra, rb in zip(a, b):
        assert ra.converged and rb.converged
        assert np.array_equal(ra.values, rb.values)
        assert ra.iterations == rb.iterations and ra.final_update == rb.final_update


def test_large_grid_path_jacobi_bit_identical(golden, oracle, ctx, monkeypatch):
    # K3b (cooperative, global memory) runs the same reference iteration
    monkeypatch.setenv("SDDG_FORCE_LARGE_SOLVER", "1")
    for name in ("ring17_t10", "running33x17_t8", "ring33_maxit"):
        kind, nx, ny, tol, mi, blend = SOLVES[name]
        w = golden[f"solve_{name}_w"]
        r = sdd.solve_dirichlet(w, nx, ny, 1.0 / (nx - 1), 1.0 / (ny - 1), _bc(oracle, kind, nx, ny, "xi"),
                                sdd.SolverConfig(tol=tol, max_iters=mi, init_blend=blend), ctx=ctx)
        info = golden[f"solve_{name}_xi_info"]
        assert np.array_equal(r.values, golden[f"solve_{name}_xi_u"])
        assert r.iterations == int(info[0]) and r.converged == bool(info[2])


def test_large_grid_rbsor_against_sparse_direct(oracle, ctx):
    # a 257^2 single-domain solve (does not fit shared memory) vs scipy spsolve
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    n = 257
    w = oracle.weight_values(B.density(B.TWOBUMP_W), UNIT, n, n)
    bc = _bc(oracle, B.TWOBUMP_W, n, n, "xi")
    r = sdd.solve_dirichlet(w, n, n, 1 / (n - 1), 1 / (n - 1), bc, sdd.SolverConfig(tol=1e-13, method="rbsor"),
                            ctx=ctx)
    assert r.converged
    h2 = (1 / (n - 1)) ** 2
    W = w.reshape(n, n)
    U = np.zeros((n, n))
    U[0, :], U[-1, :], U[:, 0], U[:, -1] = bc.bottom, bc.top, bc.left, bc.right
    m = n - 2
    idx = lambda i, j: (j - 1) * m + (i - 1)
    rows, cols, vals, rhs = [], [], [], np.zeros(m * m)
    for j in range(1, n - 1):
        for i in range(1, n - 1):
            k = idx(i, j)
            cs = {(i + 1, j): 0.5 * (W[j, i] + W[j, i + 1]), (i - 1, j): 0.5 * (W[j, i] + W[j, i - 1]),
                  (i, j + 1): 0.5 * (W[j, i] + W[j + 1, i]), (i, j - 1): 0.5 * (W[j, i] + W[j - 1, i])}
            rows.append(k); cols.append(k); vals.append(sum(cs.values()) / h2)
            for (ii, jj), c in cs.items():
                if ii in (0, n - 1) or jj in (0, n - 1):
                    rhs[k] += c / h2 * U[jj, ii]
                else:
                    rows.append(k); cols.append(idx(ii, jj)); vals.append(-c / h2)
    A = sp.csr_matrix((vals, (rows, cols)), shape=(m * m, m * m))
    U[1:-1, 1:-1] = spla.spsolve(A, rhs).reshape(m, m)
    assert np.max(np.abs(r.values - U.ravel())) <= 1e-10


def test_single_domain_513_config4_reference_solve(oracle, ctx):
    # config 4's single-domain comparison grid (513^2) goes through K3b
    n = 513
    w = oracle.weight_values(B.density(B.TWOBUMP_W), UNIT, n, n)
    res = sdd.solve_dirichlet_batch(w, n, n, 1 / 512, 1 / 512, [(0, 0, n, n)] * 2,
                                    [_bc(oracle, B.TWOBUMP_W, n, n, "xi"), _bc(oracle, B.TWOBUMP_W, n, n, "eta")],
                                    sdd.SolverConfig(tol=1e-10, method="rbsor"), ctx=ctx)
    assert all(r.converged for r in res)
    X = res[0].values.reshape(n, n)
    assert (np.diff(X, axis=1) > 0).all()   # xi strictly increasing in x (max principle per row)


def test_per_job_sor_factor_same_fixed_point_fewer_sweeps(oracle, ctx):
    # The default RB-SOR factor (omega = 0) is estimated per job from its
    # weights (a Rayleigh quotient of the Jacobi operator, solver.cu
    # sor_omega_kernel).  On config 3's shock-layer blocks the grid formula
    # (omega < 0) is far from optimal: the per-job factor must land on the
    # same fixed point (within the 1e-10 bar) in fewer sweeps for the slowest
    # job, and cost nothing on the constant-weight blocks.
    g = 1025
    w = oracle.weight_values(B.density(B.SHOCK_W), UNIT, g, g)
    rng = np.random.default_rng(5)
    subs, bcs = [], []
    for b in range(8):  # one column of blocks, crossing the shock layer
        v0, v1, v2, v3 = np.sort(rng.random(4))
        edge = lambda lo, hi: np.linspace(lo, hi, 129)  # noqa: E731
        bcs.append(sdd.EdgeData(edge(v0, v1), edge(v2, v3), edge(v0, v2), edge(v1, v3)))
        subs.append((0, b * 128, 129, 129))
    est = sdd.solve_dirichlet_batch(w, g, g, 1 / 1024, 1 / 1024, subs, bcs,
                                    sdd.SolverConfig(tol=1e-12, method="rbsor", omega=0.0), ctx=ctx)
    grid = sdd.solve_dirichlet_batch(w, g, g, 1 / 1024, 1 / 1024, subs, bcs,
                                     sdd.SolverConfig(tol=1e-12, method="rbsor", omega=-1.0), ctx=ctx)
    assert all(r.converged for r in est + grid)
    for a, b in zip(est, grid):
        assert np.max(np.abs(a.values - b.values)) <= 1e-10
    assert max(r.iterations for r in est) < 0.8 * max(r.iterations for r in grid)
    # constant weights: the estimate is the grid formula's factor
    ones = np.ones(g * g)
    e1 = sdd.solve_dirichlet_batch(ones, g, g, 1 / 1024, 1 / 1024, subs[:2], bcs[:2],
                                   sdd.SolverConfig(tol=1e-12, method="rbsor", omega=0.0), ctx=ctx)
    g1 = sdd.solve_dirichlet_batch(ones, g, g, 1 / 1024, 1 / 1024, subs[:2], bcs[:2],
                                   sdd.SolverConfig(tol=1e-12, method="rbsor", omega=-1.0), ctx=ctx)
    for a, b in zip(e1, g1):
        assert abs(a.iterations - b.iterations) <= 2
        assert np.max(np.abs(a.values - b.values)) <= 1e-10


@pytest.mark.parametrize("nx,ny", [(129, 129), (97, 130)])
def test_streamed_solver_matches_l2_solver(oracle, ctx, monkeypatch, nx, ny):
    # K3s (the packed weights streamed through a two-stage shared-memory ring
    # by cp.async.bulk + mbarriers) runs K3's iteration on the same weights:
    # identical iterates, bit for bit.  200 jobs > one per SM, so the batch
    # is not a cluster batch.
    g = 513
    w = oracle.weight_values(B.density(B.SHOCK_W), UNIT, g, g)
    rng = np.random.default_rng(nx + ny)
    subs, bcs = [], []
    for k in range(200):
        v0, v1, v2, v3 = np.sort(rng.random(4))
        ex = lambda lo, hi: np.linspace(lo, hi, nx)  # noqa: E731
        ey = lambda lo, hi: np.linspace(lo, hi, ny)  # noqa: E731
        bcs.append(sdd.EdgeData(ex(v0, v1), ex(v2, v3), ey(v0, v2), ey(v1, v3)))
        subs.append(((k * 37) % (g - nx), (k * 53) % (g - ny), nx, ny))
    cfg = sdd.SolverConfig(tol=1e-12, method="rbsor")
    monkeypatch.setenv("SDDG_SOLVER_STREAM", "1")
    a = sdd.solve_dirichlet_batch(w, g, g, 1 / (g - 1), 1 / (g - 1), subs, bcs, cfg, ctx=ctx)
    monkeypatch.delenv("SDDG_SOLVER_STREAM")
    b = sdd.solve_dirichlet_batch(w, g, g, 1 / (g - 1), 1 / (g - 1), subs, bcs, cfg, ctx=ctx)
    for ra, rb in zip(a, b):
        assert ra.converged and rb.converged
        assert np.array_equal(ra.values, rb.values)
        assert ra.iterations == rb.iterations and ra.final_update == rb.final_update

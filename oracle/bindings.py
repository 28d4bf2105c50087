"""ctypes bindings for the oracle libraries -- TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``oracle/Makefile``:

* ``Ref``   -> ``oracle/_ref/libsddref.so``: the unmodified reference library
  (/root/reference/proj/src) behind ``oracle/ref_harness.cpp``.
* ``Oracle`` -> ``oracle/_build/liboracle.so``: the plain-C restatement
  ``oracle/sdd_oracle.c``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsddref.so")
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")

# density kinds (sdd_oracle.h; same numbering as include/sddg.h)
CONSTANT, RUNNING, HUANG_SLOAN, MACKENZIE, FIVE_RING = 0, 1, 2, 3, 4
RING_W, SHOCK_W, TWOBUMP_W = 16, 17, 18
TABLE = 32

ERRORS = {1: "ValidationError", 2: "OutOfDomainError", 3: "EvaluationError",
          4: "NumericalError", 5: "LayoutError", 7: "Error"}


class Domain(C.Structure):
    _fields_ = [("xmin", C.c_double), ("xmax", C.c_double), ("ymin", C.c_double),
                ("ymax", C.c_double)]


class Density(C.Structure):
    _fields_ = [("kind", C.c_int), ("R", C.c_double), ("alpha", C.c_double),
                ("fd_h", C.c_double), ("table", C.POINTER(C.c_double)), ("tnx", C.c_int),
                ("tny", C.c_int), ("tdom", Domain)]


class WalkCfg(C.Structure):
    _fields_ = [("scheme", C.c_int), ("dt", C.c_double), ("lambda_", C.c_double),
                ("walks", C.c_int64), ("seed", C.c_uint64), ("max_steps", C.c_int64),
                ("bridge_test", C.c_int)]


class OrcBoundary(C.Structure):
    _fields_ = [("dom", Domain), ("nx", C.c_int), ("ny", C.c_int),
                ("f", C.POINTER(C.c_double) * 4), ("g", C.POINTER(C.c_double) * 4)]


PATH_DTYPE = np.dtype([("f", "<f8"), ("g", "<f8"), ("ex", "<f8"), ("ey", "<f8"),
                       ("steps", "<i8"), ("epoch", "<i4"), ("edge", "<i4")])
EST_DTYPE = np.dtype([("xi", "<f8"), ("eta", "<f8"), ("se_xi", "<f8"), ("se_eta", "<f8"),
                      ("walks", "<i8"), ("restarts", "<i8"), ("warn", "<i4"),
                      ("_pad", "<i4"), ("edge_hits", "<i8", (4,)), ("sum_f", "<f8"),
                      ("sum_g", "<f8"), ("sum_ff", "<f8"), ("sum_gg", "<f8"),
                      ("path_steps", "<i8")])


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        self.code = code
        self.kind = ERRORS.get(code, "Error")
        super().__init__(f"{self.kind}({code}) {msg}")


def density(kind, R=None, alpha=None, fd_h=1e-6):
    """Reference defaults for the builtin monitors (monitor.hpp:26-38)."""
    defaults = {CONSTANT: (1.0, 0.0), RUNNING: (15.0, 0.0), HUANG_SLOAN: (15.0, 0.7),
                MACKENZIE: (50.0, 10.0), FIVE_RING: (30.0, 0.2)}
    r0, a0 = defaults.get(kind, (0.0, 0.0))
    return Density(kind, r0 if R is None else R, a0 if alpha is None else alpha, fd_h)


def table_density(rho, dom, fd_h=1e-6):
    """A tabulated user density (rho[j, i] at the grid nodes over dom): the
    reference receives it as user_supplied(the harness's interpolant)."""
    t = np.ascontiguousarray(rho, dtype=np.float64)
    d = Density(TABLE, 0.0, 0.0, fd_h, t.ctypes.data_as(C.POINTER(C.c_double)), t.shape[1], t.shape[0],
                Domain(dom.xmin, dom.xmax, dom.ymin, dom.ymax))
    d._keep = t
    return d


def walk_cfg(scheme="linear", dt=1e-4, lam=1000.0, walks=10000, seed=1,
             max_steps=10_000_000, bridge=True):
    return WalkCfg(0 if scheme == "linear" else 1, dt, lam, walks, seed, max_steps,
                   1 if bridge else 0)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def ensure_built():
    if os.path.exists(ORACLE_SO) and (os.path.exists(REF_SO) or not os.path.isdir("/root/reference")):
        return
    subprocess.check_call(["make", "-s", "-C", HERE, "oracle"] +
                          (["ref"] if os.path.isdir("/root/reference") else []))


class Tables:
    """Eight boundary tables (f/g x bottom/top/left/right) on an nx x ny grid."""

    def __init__(self, dom, nx, ny, f, g):
        self.dom, self.nx, self.ny = dom, nx, ny
        self.f = [_f64(t) for t in f]
        self.g = [_f64(t) for t in g]

    def ptr_arrays(self):
        fa = (C.POINTER(C.c_double) * 4)(*[_dp(t) for t in self.f])
        ga = (C.POINTER(C.c_double) * 4)(*[_dp(t) for t in self.g])
        return fa, ga

    @staticmethod
    def identity(dom, nx, ny):
        """xi = x, eta = y mapped to [0,1] (BASELINE.json's boundary data)."""
        xs = np.array([dom.xmin + i * ((dom.xmax - dom.xmin) / (nx - 1)) for i in range(nx)])
        ys = np.array([dom.ymin + j * ((dom.ymax - dom.ymin) / (ny - 1)) for j in range(ny)])
        fx = (xs - dom.xmin) / (dom.xmax - dom.xmin)
        gy = (ys - dom.ymin) / (dom.ymax - dom.ymin)
        f = [fx, fx, np.zeros(ny), np.ones(ny)]
        g = [np.zeros(nx), np.ones(nx), gy, gy]
        return Tables(dom, nx, ny, f, g)


class _Lib:
    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err())

    def _err(self):
        return ""


class Ref(_Lib):
    """The reference itself (oracle/_ref/libsddref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` (needs /root/reference)")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_hardware_threads.restype = C.c_int

    def _err(self):
        return self.L.ref_last_error().decode()

    def hardware_threads(self):
        return self.L.ref_hardware_threads()

    def philox_block(self, k0, k1, c):
        cin = (C.c_uint32 * 4)(*c)
        out = (C.c_uint32 * 4)()
        self.L.ref_philox_block(C.c_uint32(k0), C.c_uint32(k1), cin, out)
        return list(out)

    def stream_u64(self, seed, pid, walk, epoch, n):
        out = np.zeros(n, np.uint64)
        self.L.ref_stream_u64(C.c_uint64(seed), C.c_uint64(pid), C.c_uint32(walk),
                              C.c_uint32(epoch), C.c_int64(n), out.ctypes.data_as(C.c_void_p))
        return out

    def stream_u01(self, seed, pid, walk, epoch, n, open_=False):
        out = np.zeros(n)
        self.L.ref_stream_u01(C.c_uint64(seed), C.c_uint64(pid), C.c_uint32(walk),
                              C.c_uint32(epoch), C.c_int64(n), C.c_int(1 if open_ else 0), _dp(out))
        return out

    def stream_normals(self, seed, pid, walk, epoch, npairs):
        out = np.zeros(2 * npairs)
        self.L.ref_stream_normals(C.c_uint64(seed), C.c_uint64(pid), C.c_uint32(walk),
                                  C.c_uint32(epoch), C.c_int64(npairs), _dp(out))
        return out

    def rho_drift(self, dens, dom, x, y):
        x, y = _f64(x), _f64(y)
        n = len(x)
        rho, bx, by = np.zeros(n), np.zeros(n), np.zeros(n)
        self._check(self.L.ref_rho_drift(C.byref(dens), C.byref(dom), C.c_int64(n), _dp(x), _dp(y),
                                         _dp(rho), _dp(bx), _dp(by)))
        return rho, bx, by

    def make_boundary(self, dens, dom, nx, ny):
        t = [np.zeros(nx), np.zeros(nx), np.zeros(ny), np.zeros(ny),
             np.zeros(nx), np.zeros(nx), np.zeros(ny), np.zeros(ny)]
        self._check(self.L.ref_make_boundary(C.byref(dens), C.byref(dom), nx, ny, *[_dp(a) for a in t]))
        return Tables(dom, nx, ny, t[:4], t[4:])

    def walk_dump(self, dens, dom, tables, cfg, px, py, pid, walk_lo, n):
        out = np.zeros(n, PATH_DTYPE)
        fa, ga = tables.ptr_arrays()
        self._check(self.L.ref_walk_dump(C.byref(dens), C.byref(dom), tables.nx, tables.ny, fa, ga,
                                         C.byref(cfg), C.c_double(px), C.c_double(py),
                                         C.c_uint64(pid), C.c_int64(walk_lo), C.c_int64(n),
                                         out.ctypes.data_as(C.c_void_p)))
        return out

    def mc_estimate_batch(self, dens, dom, tables, cfg, px, py, pid, threads=1):
        px, py = _f64(px), _f64(py)
        pid = np.ascontiguousarray(pid, dtype=np.uint64)
        n = len(px)
        out = np.zeros(n, EST_DTYPE)
        fa, ga = tables.ptr_arrays()
        self._check(self.L.ref_mc_estimate_batch(
            C.byref(dens), C.byref(dom), tables.nx, tables.ny, fa, ga, C.byref(cfg), _dp(px),
            _dp(py), pid.ctypes.data_as(C.c_void_p), C.c_int64(n), C.c_int(threads),
            out.ctypes.data_as(C.c_void_p)))
        return out

    def weight_values(self, dens, dom, nx, ny):
        w = np.zeros(nx * ny)
        self._check(self.L.ref_weight_values(C.byref(dens), C.byref(dom), nx, ny, _dp(w)))
        return w

    def solve_dirichlet(self, w, nx, ny, hx, hy, bottom, top, left, right, tol=1e-8,
                        max_iters=0, init_blend=True):
        w, bottom, top, left, right = map(_f64, (w, bottom, top, left, right))
        u = np.zeros(nx * ny)
        it, fu, cv = C.c_int64(), C.c_double(), C.c_int()
        self._check(self.L.ref_solve_dirichlet(
            _dp(w), nx, ny, C.c_double(hx), C.c_double(hy), _dp(bottom), _dp(top), _dp(left),
            _dp(right), C.c_double(tol), C.c_int64(max_iters), C.c_int(1 if init_blend else 0),
            _dp(u), C.byref(it), C.byref(fu), C.byref(cv)))
        return u, it.value, fu.value, bool(cv.value)

    def plan(self, dens, dom, nx, ny, sx, sy, strategy, k=0):
        nl = C.c_int()
        cap = sx + sy
        vert = np.zeros(cap, np.int32)
        fixed = np.zeros(cap, np.int32)
        counts = np.zeros(cap, np.int32)
        nodes = np.zeros(cap * max(nx, ny), np.int32)
        ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))
        self._check(self.L.ref_plan(C.byref(dens), C.byref(dom), nx, ny, sx, sy, strategy, k,
                                    C.byref(nl), ip(vert), ip(fixed), ip(counts), ip(nodes)))
        lines, off = [], 0
        for l in range(nl.value):
            c = int(counts[l])
            lines.append((bool(vert[l]), int(fixed[l]), nodes[off:off + c].tolist()))
            off += c
        return lines

    def solve_interfaces(self, dens, dom, nx, ny, sx, sy, strategy, k, tables, cfg, threads=0):
        n_lines = (sx - 1) + (sy - 1)
        lens = [ny] * (sx - 1) + [nx] * (sy - 1)
        tot = sum(lens)
        xi, eta, sxi, seta = (np.zeros(tot) for _ in range(4))
        mc, rs = C.c_int64(), C.c_int64()
        fa, ga = tables.ptr_arrays()
        self._check(self.L.ref_solve_interfaces(
            C.byref(dens), C.byref(dom), nx, ny, sx, sy, strategy, k, fa, ga, C.byref(cfg),
            C.c_int(threads), _dp(xi), _dp(eta), _dp(sxi), _dp(seta), C.byref(mc), C.byref(rs)))
        out, off = [], 0
        for l in range(n_lines):
            out.append((xi[off:off + lens[l]], eta[off:off + lens[l]], sxi[off:off + lens[l]],
                        seta[off:off + lens[l]]))
            off += lens[l]
        return out, mc.value, rs.value

    def invert_mesh(self, xi, eta, nx, ny, dom, m_xi, m_eta, threads=1):
        xi, eta = _f64(xi), _f64(eta)
        x, y = np.zeros(m_xi * m_eta), np.zeros(m_xi * m_eta)
        self._check(self.L.ref_invert_mesh(_dp(xi), _dp(eta), nx, ny, C.byref(dom), m_xi, m_eta,
                                           threads, _dp(x), _dp(y)))
        return x, y

    def quality(self, x, y, m_xi, m_eta, dom, ref_x=None, ref_y=None, dens=None):
        x, y = _f64(x), _f64(y)
        out = np.zeros(5)
        rx = _dp(_f64(ref_x)) if ref_x is not None else None
        ry = _dp(_f64(ref_y)) if ref_y is not None else None
        keep = (ref_x, ref_y)
        self._check(self.L.ref_quality(_dp(x), _dp(y), m_xi, m_eta, C.byref(dom), rx, ry,
                                       C.byref(dens) if dens is not None else None, _dp(out)))
        del keep
        return out

    def perona_malik(self, xi, eta, nx, ny, dom, k, dt, steps, scope=0, sx=1, sy=1):
        xi, eta = _f64(xi).copy(), _f64(eta).copy()
        self._check(self.L.ref_perona_malik(_dp(xi), _dp(eta), nx, ny, C.byref(dom), C.c_double(k),
                                            C.c_double(dt), steps, scope, sx, sy))
        return xi, eta

    def smooth_interface(self, v, span):
        v = _f64(v)
        out = np.zeros_like(v)
        self._check(self.L.ref_smooth_interface(_dp(v), len(v), span, _dp(out)))
        return out

    def solve_sdd_smoothed(self, dens, dom, nx, ny, sx, sy, strategy, k, cfg, tol, span):
        xi, eta = np.zeros(nx * ny), np.zeros(nx * ny)
        self._check(self.L.ref_solve_sdd_smoothed(C.byref(dens), C.byref(dom), nx, ny, sx, sy, strategy,
                                                  k, C.byref(cfg), C.c_double(tol), span, _dp(xi), _dp(eta)))
        return xi, eta

    def write_mesh(self, x, y, m_xi, m_eta, xi, eta, nx, ny, path):
        x, y, xi, eta = map(_f64, (x, y, xi, eta))
        self._check(self.L.ref_write_mesh(_dp(x), _dp(y), m_xi, m_eta, _dp(xi), _dp(eta), nx, ny,
                                          path.encode()))

    def solve_single_domain(self, dens, dom, nx, ny, tol=1e-8):
        xi, eta = np.zeros(nx * ny), np.zeros(nx * ny)
        self._check(self.L.ref_solve_single_domain(C.byref(dens), C.byref(dom), nx, ny,
                                                   C.c_double(tol), _dp(xi), _dp(eta)))
        return xi, eta

    def solve_sdd(self, dens, dom, nx, ny, sx, sy, strategy, k, cfg, tol=1e-8, max_iters=0,
                  threads=0):
        xi, eta, t = np.zeros(nx * ny), np.zeros(nx * ny), np.zeros(3)
        self._check(self.L.ref_solve_sdd(C.byref(dens), C.byref(dom), nx, ny, sx, sy, strategy, k,
                                         C.byref(cfg), C.c_double(tol), C.c_int64(max_iters),
                                         C.c_int(threads), _dp(xi), _dp(eta), _dp(t)))
        return xi, eta, t


class Oracle(_Lib):
    """The plain-C restatement (oracle/_build/liboracle.so)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.L = C.CDLL(path)
        L.orc_rho.restype = C.c_double
        L.orc_table_at.restype = C.c_double
        L.orc_bd_value.restype = C.c_double
        L.orc_w_formula.restype = C.c_double
        L.orc_w_formula.argtypes = [C.c_int, C.c_double, C.c_double]

    def _bd(self, tables):
        fa, ga = tables.ptr_arrays()
        b = OrcBoundary(tables.dom, tables.nx, tables.ny, fa, ga)
        b._keep = tables
        return b

    def philox_block(self, k0, k1, c):
        cin = (C.c_uint32 * 4)(*c)
        out = (C.c_uint32 * 4)()
        self.L.orc_philox_block(C.c_uint32(k0), C.c_uint32(k1), cin, out)
        return list(out)

    def stream_u64(self, seed, pid, walk, epoch, n):
        out = np.zeros(n, np.uint64)
        self.L.orc_stream_u64(C.c_uint64(seed), C.c_uint64(pid), C.c_uint32(walk),
                              C.c_uint32(epoch), C.c_int64(n), out.ctypes.data_as(C.c_void_p))
        return out

    def stream_normals(self, seed, pid, walk, epoch, npairs):
        out = np.zeros(2 * npairs)
        self.L.orc_stream_normals(C.c_uint64(seed), C.c_uint64(pid), C.c_uint32(walk),
                                  C.c_uint32(epoch), C.c_int64(npairs), _dp(out))
        return out

    def w(self, kind, x, y):
        return self.L.orc_w_formula(kind, x, y)

    def rho_drift(self, dens, x, y):
        x, y = _f64(x), _f64(y)
        rho, bx, by = np.zeros(len(x)), np.zeros(len(x)), np.zeros(len(x))
        b1, b2 = C.c_double(), C.c_double()
        for k in range(len(x)):
            rho[k] = self.L.orc_rho(C.byref(dens), C.c_double(x[k]), C.c_double(y[k]))
            self._check(self.L.orc_drift(C.byref(dens), C.c_double(x[k]), C.c_double(y[k]),
                                         C.byref(b1), C.byref(b2)))
            bx[k], by[k] = b1.value, b2.value
        return rho, bx, by

    def solve_1d_boundary(self, dens, dom, nx, ny, edge):
        n = nx if edge in (0, 1) else ny
        out = np.zeros(n)
        self.L.orc_solve_1d_boundary(C.byref(dens), C.byref(dom), nx, ny, edge, _dp(out))
        return out

    def make_boundary(self, dens, dom, nx, ny):
        b = [self.solve_1d_boundary(dens, dom, nx, ny, e) for e in range(4)]
        f = [b[0], b[1], np.zeros(ny), np.ones(ny)]
        g = [np.zeros(nx), np.ones(nx), b[2], b[3]]
        return Tables(dom, nx, ny, f, g)

    def walk_dump(self, dens, dom, tables, cfg, px, py, pid, walk_lo, n):
        out = np.zeros(n, PATH_DTYPE)
        bd = self._bd(tables)
        self._check(self.L.orc_walk_dump(C.byref(dens), C.byref(dom), C.byref(bd), C.byref(cfg),
                                         C.c_double(px), C.c_double(py), C.c_uint64(pid),
                                         C.c_int64(walk_lo), C.c_int64(n),
                                         out.ctypes.data_as(C.c_void_p)))
        return out

    def mc_estimate_batch(self, dens, dom, tables, cfg, px, py, pid, threads=1):
        px, py = _f64(px), _f64(py)
        pid = np.ascontiguousarray(pid, dtype=np.uint64)
        out = np.zeros(len(px), EST_DTYPE)
        bd = self._bd(tables)
        self._check(self.L.orc_mc_estimate_batch(
            C.byref(dens), C.byref(dom), C.byref(bd), C.byref(cfg), _dp(px), _dp(py),
            pid.ctypes.data_as(C.c_void_p), C.c_int64(len(px)), C.c_int(threads),
            out.ctypes.data_as(C.c_void_p)))
        return out

    def weight_values(self, dens, dom, nx, ny):
        w = np.zeros(nx * ny)
        self.L.orc_weight_values(C.byref(dens), C.byref(dom), nx, ny, _dp(w))
        return w

    def solve_dirichlet(self, w, nx, ny, hx, hy, bottom, top, left, right, tol=1e-8,
                        max_iters=0, init_blend=True):
        w, bottom, top, left, right = map(_f64, (w, bottom, top, left, right))
        u = np.zeros(nx * ny)
        it, fu, cv = C.c_int64(), C.c_double(), C.c_int()
        self._check(self.L.orc_solve_dirichlet(
            _dp(w), nx, ny, C.c_double(hx), C.c_double(hy), _dp(bottom), _dp(top), _dp(left),
            _dp(right), C.c_double(tol), C.c_int64(max_iters), C.c_int(1 if init_blend else 0),
            _dp(u), C.byref(it), C.byref(fu), C.byref(cv)))
        return u, it.value, fu.value, bool(cv.value)

    def plan_line(self, strategy, k, dens, dom, nx, ny, vertical, fixed):
        out = np.zeros(max(nx, ny), np.int32)
        n = self.L.orc_plan_line(strategy, k, C.byref(dens), C.byref(dom), nx, ny,
                                 1 if vertical else 0, fixed, out.ctypes.data_as(C.POINTER(C.c_int)))
        if n < 0:
            raise OracleError(1, "equispaced count out of range")
        return out[:n].tolist()

    def fill_line(self, n, known_pos, known_xi, known_eta):
        kp = np.ascontiguousarray(known_pos, dtype=np.int32)
        kx, ke = _f64(known_xi), _f64(known_eta)
        xi, eta = np.zeros(n), np.zeros(n)
        self.L.orc_fill_line(n, kp.ctypes.data_as(C.POINTER(C.c_int)), _dp(kx), _dp(ke),
                             len(kp), _dp(xi), _dp(eta))
        return xi, eta

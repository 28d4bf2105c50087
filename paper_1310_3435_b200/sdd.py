"""Python mirror of the reference ``sdd::`` API for the hot path, over the
C-ABI in ``include/sddg.h`` (library ``_lib/libsddg.so``).

Names, argument meaning and error classes follow the reference
(/root/reference/proj/include/sdd/*.hpp) so tests read like the reference's
own tests:

=====================================  ==========================================
reference (C++)                        here
=====================================  ==========================================
``MonitorFunction`` (monitor.hpp)      :class:`MonitorFunction` (data descriptor)
``RectDomain``/``GridSpec``            :class:`RectDomain`, :class:`GridSpec`
``WalkConfig`` (sde.hpp:16-26)         :class:`WalkConfig` (+ ``precision``)
``mc_estimate`` (sde.hpp:75-77)        :func:`mc_estimate`, :func:`mc_estimate_batch`
``make_boundary_data`` (boundary.hpp)  :func:`make_boundary_data`
``SolverConfig``/``solve_dirichlet``   :class:`SolverConfig`, :func:`solve_dirichlet`
``build_layout``/``plan_interface_points`` :func:`build_layout`, :func:`plan_interface_points`
``solve_interfaces``/``solve_sdd``     :func:`solve_interfaces`, :func:`solve_sdd`
=====================================  ==========================================

All compute runs on the B200 through the library; if the library or the GPU
is missing the calls raise -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field

import numpy as np

_LIB_PATH = os.environ.get("SDDG_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libsddg.so")


# --------------------------------------------------------------- errors
class Error(RuntimeError):
    """sdd::Error (proj/include/sdd/errors.hpp:8-11)."""


class ValidationError(Error): ...
class OutOfDomainError(Error): ...
class EvaluationError(Error): ...
class NumericalError(Error): ...
class LayoutError(Error): ...
class CudaError(Error): ...
class InversionError(Error): ...
class TanglingError(Error): ...


_ERR = {1: ValidationError, 2: OutOfDomainError, 3: EvaluationError, 4: NumericalError,
        5: LayoutError, 6: CudaError, 7: Error, 8: InversionError, 9: TanglingError}

# --------------------------------------------------------------- C structs
CONSTANT, RUNNING, HUANG_SLOAN, MACKENZIE, FIVE_RING = 0, 1, 2, 3, 4
RING_W, SHOCK_W, TWOBUMP_W = 16, 17, 18
TABLE = 32
GRAD_REFERENCE, GRAD_ANALYTIC = 0, 1
LINEAR, EXPONENTIAL = 0, 1
FP64, FP32 = 0, 1
JACOBI, RBSOR = 0, 1
PLACE = {"all": 0, "equispaced": 1, "optimal": 2, "equidistributed": 3}
INTERP = {"linear": 0, "spline": 1}
BC_REFERENCE, BC_IDENTITY = 0, 1


class _Domain(C.Structure):
    _fields_ = [("xmin", C.c_double), ("xmax", C.c_double), ("ymin", C.c_double),
                ("ymax", C.c_double)]


class _Density(C.Structure):
    _fields_ = [("kind", C.c_int32), ("grad_mode", C.c_int32), ("R", C.c_double),
                ("alpha", C.c_double), ("fd_h", C.c_double), ("table", C.POINTER(C.c_double)),
                ("tnx", C.c_int32), ("tny", C.c_int32), ("tdom", _Domain)]


class _Boundary(C.Structure):
    _fields_ = [("dom", _Domain), ("nx", C.c_int32), ("ny", C.c_int32),
                ("f", C.POINTER(C.c_double) * 4), ("g", C.POINTER(C.c_double) * 4)]


class _WalkCfg(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("precision", C.c_int32), ("dt", C.c_double),
                ("lambda_", C.c_double), ("walks", C.c_int64), ("seed", C.c_uint64),
                ("max_steps", C.c_int64), ("bridge_test", C.c_int32), ("form", C.c_int32)]


class _SolverCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int64), ("init_blend", C.c_int32),
                ("method", C.c_int32), ("omega", C.c_double)]


class _Subdomain(C.Structure):
    _fields_ = [("i0", C.c_int32), ("j0", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32)]


class _SddStats(C.Structure):
    _fields_ = [("t_bd", C.c_double), ("t_stoc", C.c_double), ("t_sub", C.c_double),
                ("t_smooth", C.c_double), ("mc_points", C.c_int64),
                ("subdomain_solves", C.c_int64), ("restarts", C.c_int64),
                ("path_steps", C.c_int64), ("warnings", C.c_int32), ("reserved", C.c_int32)]


ESTIMATE_DTYPE = np.dtype([("xi", "<f8"), ("eta", "<f8"), ("se_xi", "<f8"), ("se_eta", "<f8"),
                           ("walks", "<i8"), ("restarts", "<i8"), ("warn", "<i4"),
                           ("reserved", "<i4"), ("edge_hits", "<i8", (4,)), ("sum_f", "<f8"),
                           ("sum_g", "<f8"), ("sum_ff", "<f8"), ("sum_gg", "<f8"),
                           ("path_steps", "<i8")])
PATH_DTYPE = np.dtype([("f", "<f8"), ("g", "<f8"), ("ex", "<f8"), ("ey", "<f8"),
                       ("steps", "<i8"), ("epoch", "<i4"), ("edge", "<i4")])
SOLVE_INFO_DTYPE = np.dtype([("iterations", "<i8"), ("final_update", "<f8"),
                             ("converged", "<i4"), ("reserved", "<i4")])
assert ESTIMATE_DTYPE.itemsize == 128 and PATH_DTYPE.itemsize == 48

_lib = None
_lib_lock = threading.Lock()


def library_path():
    return _LIB_PATH


def lib():
    """Load libsddg.so (raises if the sm_100a extension was not built)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise ImportError(f"{_LIB_PATH} not built: run __graft_entry__.build() or "
                                  "python paper_1310_3435_b200/build.py")
            # multi-GPU contexts load NCCL at run time: point the library at
            # PyTorch's bundled libnccl.so.2 (the copy torch links), so the
            # two never load different copies of the same soname
            if "SDDG_NCCL_PATH" not in os.environ:
                try:
                    import importlib.util
                    spec = importlib.util.find_spec("nvidia.nccl")
                    for d in (spec.submodule_search_locations or []) if spec else []:
                        cand = os.path.join(d, "lib", "libnccl.so.2")
                        if os.path.exists(cand):
                            os.environ["SDDG_NCCL_PATH"] = cand
                            break
                except (ImportError, ValueError):
                    pass
            L = C.CDLL(_LIB_PATH)
            L.sddg_version.restype = C.c_char_p
            L.sddg_last_error.restype = C.c_char_p
            L.sddg_last_error.argtypes = [C.c_void_p]
            L.sddg_create.argtypes = [C.c_int32, C.POINTER(C.c_void_p)]
            L.sddg_destroy.argtypes = [C.c_void_p]
            _lib = L
        return _lib


def _check(rc, ctx=None):
    if rc != 0:
        msg = lib().sddg_last_error(ctx).decode() if ctx is not None else lib().sddg_last_error(None).decode()
        raise _ERR.get(rc, Error)(msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# --------------------------------------------------------------- context
class NcclId(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 128)]


def nccl_unique_id() -> bytes:
    """sddg_nccl_unique_id: rank 0 creates it and hands it to the other ranks."""
    i = NcclId()
    _check(lib().sddg_nccl_unique_id(C.byref(i)))
    return bytes(i.bytes)


class Context:
    """One device, its stream and buffers (sddg_create / sddg_destroy); or
    several GPUs (Context.dist: one process per GPU over NCCL;
    Context.multi: one process driving several devices)."""

    def __init__(self, device=0, _handle=None):
        self._h = C.c_void_p()
        if _handle is None:
            _check(lib().sddg_create(int(device), C.byref(self._h)))
        else:
            self._h = _handle
        self.device = device

    @staticmethod
    def dist(device: int, rank: int, nranks: int, nccl_id: bytes) -> "Context":
        """sddg_create_dist: this process is `rank` of `nranks` (collective)."""
        h = C.c_void_p()
        i = NcclId()
        C.memmove(i.bytes, nccl_id, 128)
        _check(lib().sddg_create_dist(int(device), int(rank), int(nranks), C.byref(i), C.byref(h)))
        return Context(device, _handle=h)

    @staticmethod
    def multi(devices) -> "Context":
        """sddg_create_multi: one process drives every device in `devices`."""
        devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        _check(lib().sddg_create_multi(len(devices), devs, C.byref(h)))
        return Context(int(devices[0]), _handle=h)

    def team_info(self):
        r, n, loc, nc = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().sddg_team_info(self._h, C.byref(r), C.byref(n), C.byref(loc), C.byref(nc)), self._h)
        return {"rank": r.value, "nranks": n.value, "local_devices": loc.value, "nccl": bool(nc.value)}

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().sddg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def probe_fma_peak(self, precision="fp64"):
        """Measured non-tensor FMA peak (TFLOP/s) of this device."""
        t = C.c_double()
        _check(lib().sddg_probe_fma_peak(self._h, FP64 if precision == "fp64" else FP32, C.byref(t)),
               self._h)
        return t.value

    def probe_onchip_bandwidth(self):
        """Measured L2 and shared-memory read bandwidth (GB/s) of this device."""
        l2, sm = C.c_double(), C.c_double()
        _check(lib().sddg_probe_onchip_bandwidth(self._h, C.byref(l2), C.byref(sm)), self._h)
        return {"l2_GBps": l2.value, "smem_GBps": sm.value}

    def last_stats(self):
        s, n, ms = C.c_int64(), C.c_int64(), C.c_double()
        _check(lib().sddg_last_stats(self._h, C.byref(s), C.byref(n), C.byref(ms)), self._h)
        h, tms = C.c_int64(), C.c_double()
        _check(lib().sddg_last_tail_stats(self._h, C.byref(h), C.byref(tms)), self._h)
        return {"path_steps": s.value, "launches": n.value, "kernel_ms": ms.value,
                "tail_handoffs": h.value, "tail_ms": tms.value}


_default_ctx = {}


def default_context(device=None):
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


# --------------------------------------------------------------- geometry
@dataclass(frozen=True)
class RectDomain:
    """sdd::RectDomain (proj/include/sdd/geometry.hpp:27-46)."""
    xmin: float
    xmax: float
    ymin: float
    ymax: float

    def __post_init__(self):
        if not (self.xmin < self.xmax) or not (self.ymin < self.ymax):
            raise ValidationError("RectDomain: requires xmin < xmax and ymin < ymax")

    def strictly_inside(self, x, y):
        return self.xmin < x < self.xmax and self.ymin < y < self.ymax

    def c(self):
        return _Domain(self.xmin, self.xmax, self.ymin, self.ymax)


@dataclass(frozen=True)
class GridSpec:
    """sdd::GridSpec (geometry.hpp:49-70): index (i, j) -> j*nx + i."""
    domain: RectDomain
    nx: int
    ny: int

    def __post_init__(self):
        if self.nx < 3 or self.ny < 3:
            raise ValidationError(f"GridSpec: needs nx >= 3 and ny >= 3, got {self.nx}x{self.ny}")

    def hx(self):
        return (self.domain.xmax - self.domain.xmin) / (self.nx - 1)

    def hy(self):
        return (self.domain.ymax - self.domain.ymin) / (self.ny - 1)

    def idx(self, i, j):
        return j * self.nx + i

    def node(self, i, j):
        return (self.domain.xmin + i * self.hx(), self.domain.ymin + j * self.hy())


# --------------------------------------------------------------- density
@dataclass(frozen=True)
class MonitorFunction:
    """Data form of sdd::MonitorFunction (proj/include/sdd/monitor.hpp:23-70)."""
    kind: int
    R: float = 0.0
    alpha: float = 0.0
    grad_mode: int = GRAD_REFERENCE
    fd_h: float = 1e-6
    domain: RectDomain = RectDomain(0.0, 1.0, 0.0, 1.0)
    # SDDG_DENS_TABLE: rho samples (ny, nx) at the grid nodes over `domain`
    table: np.ndarray | None = field(default=None, compare=False, hash=False, repr=False)

    @staticmethod
    def constant(value=1.0):
        return MonitorFunction(CONSTANT, R=value)

    @staticmethod
    def running_example(R=15.0):
        return MonitorFunction(RUNNING, R=R)

    @staticmethod
    def huang_sloan(alpha=0.7, R=15.0):
        return MonitorFunction(HUANG_SLOAN, R=R, alpha=alpha)

    @staticmethod
    def mackenzie(alpha=10.0, R=50.0):
        return MonitorFunction(MACKENZIE, R=R, alpha=alpha)

    @staticmethod
    def five_ring(alpha=0.2, R=30.0, analytic=False):
        """analytic=True: performance mode (fastmath tanh, drift as
        -alpha J grad u / rho^2), checked statistically against the reference."""
        return MonitorFunction(FIVE_RING, R=R, alpha=alpha,
                               grad_mode=GRAD_ANALYTIC if analytic else GRAD_REFERENCE,
                               domain=RectDomain(-1.0, 1.0, -1.0, 1.0))

    @staticmethod
    def by_name(name, R=None, alpha=None):
        """MonitorFunction::by_name (proj/src/monitor.cpp:82-103) + BASELINE densities."""
        if name == "constant":
            return MonitorFunction.constant(1.0 if R is None else R)
        if name in ("running", "running-example"):
            return MonitorFunction.running_example(15.0 if R is None else R)
        if name == "huang-sloan":
            return MonitorFunction.huang_sloan(0.7 if alpha is None else alpha, 15.0 if R is None else R)
        if name == "mackenzie":
            return MonitorFunction.mackenzie(10.0 if alpha is None else alpha, 50.0 if R is None else R)
        if name == "five-ring":
            return MonitorFunction.five_ring(0.2 if alpha is None else alpha, 30.0 if R is None else R)
        if name in ("ring", "shock", "two-bump"):
            return MonitorFunction.weight({"ring": RING_W, "shock": SHOCK_W, "two-bump": TWOBUMP_W}[name])
        raise ValidationError(f"unknown monitor '{name}'")

    @staticmethod
    def weight(kind, analytic=False, fd_step=1e-6, domain=RectDomain(0.0, 1.0, 0.0, 1.0)):
        """A BASELINE density given as w; the reference sees user_supplied(rho=1/w)
        (monitor.cpp:73-80).  analytic=True uses grad(w)/w instead of the FD."""
        return MonitorFunction(kind, grad_mode=GRAD_ANALYTIC if analytic else GRAD_REFERENCE,
                               fd_h=fd_step, domain=domain)

    @staticmethod
    def tabulated(rho, domain: RectDomain, analytic=False, fd_step=1e-6):
        """Any user_supplied density as data (SDDG_DENS_TABLE): rho sampled at
        the nodes of a grid over `domain`, rho[j, i] at (x_i, y_j), read through
        the library's Catmull-Rom bicubic interpolant.  analytic=False: the
        reference's central difference of the interpolant (bit-faithful to
        MonitorFunction::user_supplied of that interpolant); analytic=True:
        its exact gradient (performance mode, fp64 or fp32)."""
        t = np.ascontiguousarray(rho, dtype=np.float64)
        if t.ndim != 2 or t.shape[0] < 2 or t.shape[1] < 2:
            raise ValidationError("tabulated density: rho must be a 2-D array of at least 2 x 2")
        return MonitorFunction(TABLE, grad_mode=GRAD_ANALYTIC if analytic else GRAD_REFERENCE,
                               fd_h=fd_step, domain=domain, table=t)

    ring = staticmethod(lambda analytic=False: MonitorFunction.weight(RING_W, analytic))
    shock = staticmethod(lambda analytic=False: MonitorFunction.weight(SHOCK_W, analytic))
    two_bump = staticmethod(lambda analytic=False: MonitorFunction.weight(TWOBUMP_W, analytic))

    def with_grad(self, grad_mode):
        return MonitorFunction(self.kind, self.R, self.alpha, grad_mode, self.fd_h, self.domain, self.table)

    def c(self):
        d = _Density(self.kind, self.grad_mode, self.R, self.alpha, self.fd_h)
        if self.table is not None:
            d.table = self.table.ctypes.data_as(C.POINTER(C.c_double))
            d.tny, d.tnx = self.table.shape
            d.tdom = self.domain.c()
            d._keep = self.table
        return d


# --------------------------------------------------------------- configs
@dataclass
class WalkConfig:
    """sdd::WalkConfig (proj/include/sdd/sde.hpp:16-26); defaults as the reference."""
    scheme: str = "exponential"
    dt: float = 1e-4
    lambda_: float = 1000.0
    walks: int = 10000
    seed: int = 0
    max_steps: int = 10_000_000
    bridge_test: bool = True
    precision: str = "fp64"
    form: str = "reference"  # "literal": BASELINE's dX = grad(w) dt + sqrt(2w) dW (SDDG_FORM_LITERAL)

    def c(self):
        sch = {"linear": LINEAR, "exponential": EXPONENTIAL}.get(self.scheme, 99)
        prec = {"fp64": FP64, "fp32": FP32}.get(self.precision, 99)
        form = {"reference": 0, "literal": 1}.get(self.form, 99)
        return _WalkCfg(sch, prec, self.dt, self.lambda_, int(self.walks), int(self.seed),
                        int(self.max_steps), 1 if self.bridge_test else 0, form)


@dataclass
class SolverConfig:
    """sdd::SolverConfig (proj/include/sdd/detsolver.hpp:11-18) + method."""
    tol: float = 1e-8
    max_iters: int = 0
    init_blend: bool = True
    method: str = "jacobi"
    omega: float = 0.0

    def c(self):
        m = {"jacobi": JACOBI, "rbsor": RBSOR, "sor": RBSOR}.get(self.method, 99)
        return _SolverCfg(self.tol, int(self.max_iters), 1 if self.init_blend else 0, m, self.omega)


# --------------------------------------------------------------- boundary data
@dataclass
class EdgeData:
    """sdd::EdgeData (detsolver.hpp:21-23)."""
    bottom: np.ndarray
    top: np.ndarray
    left: np.ndarray
    right: np.ndarray

    def arrays(self):
        return [self.bottom, self.top, self.left, self.right]


@dataclass
class BoundaryData:
    """sdd::BoundaryData (boundary.hpp:12-18)."""
    spec: GridSpec
    f: EdgeData
    g: EdgeData

    def c(self):
        self._keep = [_f64(a) for a in self.f.arrays() + self.g.arrays()]
        fa = (C.POINTER(C.c_double) * 4)(*[_dp(a) for a in self._keep[:4]])
        ga = (C.POINTER(C.c_double) * 4)(*[_dp(a) for a in self._keep[4:]])
        return _Boundary(self.spec.domain.c(), self.spec.nx, self.spec.ny, fa, ga)


def make_boundary_data(m: MonitorFunction, spec: GridSpec, mode=BC_REFERENCE) -> BoundaryData:
    """sdd::make_boundary_data (proj/src/boundary.cpp:44-56); mode BC_IDENTITY gives
    xi = x, eta = y (BASELINE.json)."""
    nx, ny = spec.nx, spec.ny
    t = [np.zeros(n) for n in (nx, nx, ny, ny, nx, nx, ny, ny)]
    arr = (C.POINTER(C.c_double) * 8)(*[_dp(a) for a in t])
    d, dom = m.c(), spec.domain.c()
    _check(lib().sddg_make_boundary_data(C.byref(d), C.byref(dom), nx, ny, mode, arr))
    return BoundaryData(spec, EdgeData(*t[:4]), EdgeData(*t[4:]))


# --------------------------------------------------------------- walks
@dataclass
class McEstimate:
    """sdd::McEstimate (sde.hpp:61-68)."""
    xi: float
    eta: float
    stderr_xi: float
    stderr_eta: float
    walks: int
    restarts: int
    reliability_warning: bool
    edge_hits: list
    path_steps: int = 0  # executed steps of the node's walks, all epochs (not in the reference)

    @staticmethod
    def from_record(r):
        return McEstimate(float(r["xi"]), float(r["eta"]), float(r["se_xi"]), float(r["se_eta"]),
                          int(r["walks"]), int(r["restarts"]), bool(r["warn"]),
                          [int(v) for v in r["edge_hits"]], int(r["path_steps"]))


def mc_estimate_batch(points, point_ids, m: MonitorFunction, domain: RectDomain,
                      bd: BoundaryData, cfg: WalkConfig, ctx: Context | None = None) -> np.ndarray:
    """Batched sdd::mc_estimate: returns an ESTIMATE_DTYPE record per point."""
    ctx = ctx or default_context()
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
    px, py = _f64(pts[:, 0]), _f64(pts[:, 1])
    pid = np.ascontiguousarray(point_ids, dtype=np.uint64)
    if len(pid) != len(px):
        raise ValidationError("point_ids length mismatch")
    out = np.zeros(len(px), ESTIMATE_DTYPE)
    d, dom, b, c = m.c(), domain.c(), bd.c(), cfg.c()
    _check(lib().sddg_mc_estimate_batch(ctx.handle, C.byref(d), C.byref(dom), C.byref(b), C.byref(c),
                                        _dp(px), _dp(py), pid.ctypes.data_as(C.c_void_p),
                                        C.c_int64(len(px)), out.ctypes.data_as(C.c_void_p)), ctx.handle)
    return out


def mc_estimate(p, point_id, m, domain, bd, cfg, ctx=None) -> McEstimate:
    """sdd::mc_estimate (proj/include/sdd/sde.hpp:75-77)."""
    return McEstimate.from_record(mc_estimate_batch([p], [point_id], m, domain, bd, cfg, ctx)[0])


def mc_estimate_batch_device(px, py, pid, out, m, domain, bd, cfg, ctx=None, stream=None):
    """Device-resident variant: px, py (float64), pid (int64/uint64) and out
    (uint8 tensor of n*128 bytes) are CUDA tensors; stream a torch stream."""
    ctx = ctx or default_context()
    d, dom, b, c = m.c(), domain.c(), bd.c(), cfg.c()
    st = C.c_void_p(stream.cuda_stream if stream is not None else 0)
    _check(lib().sddg_mc_estimate_batch_device(
        ctx.handle, C.byref(d), C.byref(dom), C.byref(b), C.byref(c), C.c_void_p(px.data_ptr()),
        C.c_void_p(py.data_ptr()), C.c_void_p(pid.data_ptr()), C.c_int64(px.numel()),
        C.c_void_p(out.data_ptr()), st), ctx.handle)


class _IpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64)]


class PeerGather:
    """A device gather buffer of n_total ESTIMATE records that other ranks
    (processes) open through CUDA IPC and write into directly
    (sddg_gather_alloc/open/close/free/read)."""

    def __init__(self, n_total: int, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.n_total = int(n_total)
        self.ptr = C.c_void_p()
        h = _IpcHandle()
        _check(lib().sddg_gather_alloc(self.ctx.handle, C.c_int64(self.n_total), C.byref(self.ptr),
                                       C.byref(h)), self.ctx.handle)
        self.handle = bytes(h.bytes)
        self._opened = []

    def open(self, handle: bytes) -> int:
        """Map a peer's buffer; returns its device address in this process."""
        h = _IpcHandle()
        C.memmove(h.bytes, handle, 64)
        p = C.c_void_p()
        _check(lib().sddg_gather_open(self.ctx.handle, C.byref(h), C.byref(p)), self.ctx.handle)
        self._opened.append(p)
        return p.value

    def read(self) -> np.ndarray:
        out = np.zeros(self.n_total, ESTIMATE_DTYPE)
        _check(lib().sddg_gather_read(self.ctx.handle, self.ptr, C.c_int64(self.n_total),
                                      out.ctypes.data_as(C.c_void_p)), self.ctx.handle)
        return out

    def close(self):
        for p in self._opened:
            _check(lib().sddg_gather_close(self.ctx.handle, p), self.ctx.handle)
        self._opened = []
        if self.ptr:
            _check(lib().sddg_gather_free(self.ctx.handle, self.ptr), self.ctx.handle)
            self.ptr = C.c_void_p()


def mc_estimate_gather(points, point_ids, global_index, peer_ptrs, n_total, m, domain, bd, cfg,
                       ctx=None):
    """mc_estimate_batch whose records K2 stores at slot global_index[k] of
    every buffer in peer_ptrs (device addresses valid in this process)."""
    ctx = ctx or default_context()
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
    px, py = _f64(pts[:, 0]), _f64(pts[:, 1])
    pid = np.ascontiguousarray(point_ids, dtype=np.uint64)
    gi = np.ascontiguousarray(global_index, dtype=np.int64)
    if len(pid) != len(px) or len(gi) != len(px):
        raise ValidationError("point_ids / global_index length mismatch")
    peers = (C.c_void_p * len(peer_ptrs))(*[C.c_void_p(int(p)) for p in peer_ptrs])
    d, dom, b, c = m.c(), domain.c(), bd.c(), cfg.c()
    _check(lib().sddg_mc_estimate_gather(ctx.handle, C.byref(d), C.byref(dom), C.byref(b), C.byref(c),
                                         _dp(px), _dp(py), pid.ctypes.data_as(C.c_void_p),
                                         gi.ctypes.data_as(C.c_void_p), C.c_int64(len(px)), peers,
                                         C.c_int32(len(peer_ptrs)), C.c_int64(n_total)), ctx.handle)


def walk_dump(p, point_id, m, domain, bd, cfg, walk_lo=0, n=1, ctx=None) -> np.ndarray:
    """Per-path (f, g, exit point, steps, epoch, edge) of walks [walk_lo, walk_lo+n)."""
    ctx = ctx or default_context()
    out = np.zeros(n, PATH_DTYPE)
    d, dom, b, c = m.c(), domain.c(), bd.c(), cfg.c()
    _check(lib().sddg_walk_dump(ctx.handle, C.byref(d), C.byref(dom), C.byref(b), C.byref(c),
                                C.c_double(p[0]), C.c_double(p[1]), C.c_uint64(point_id),
                                C.c_int64(walk_lo), C.c_int64(n), out.ctypes.data_as(C.c_void_p)),
           ctx.handle)
    return out


# --------------------------------------------------------------- solver
@dataclass
class SolveResult:
    """sdd::SolveResult (detsolver.hpp:25-31)."""
    values: np.ndarray
    iterations: int
    final_update: float
    converged: bool
    warning: str = ""


def solve_dirichlet_batch(w_global, gnx, gny, hx, hy, subdomains, bcs, cfg: SolverConfig,
                          ctx=None):
    """Batched sdd::solve_dirichlet.  subdomains: [(i0, j0, nx, ny)], bcs: [EdgeData]."""
    ctx = ctx or default_context()
    w = _f64(w_global)
    subs = (_Subdomain * len(subdomains))(*[_Subdomain(*s) for s in subdomains])
    packed = _f64(np.concatenate([np.concatenate([_f64(a) for a in e.arrays()]) for e in bcs])) \
        if bcs else np.zeros(0)
    total = sum(s[2] * s[3] for s in subdomains)
    u = np.zeros(total)
    info = np.zeros(len(subdomains), SOLVE_INFO_DTYPE)
    sc = cfg.c()
    _check(lib().sddg_solve_dirichlet_batch(ctx.handle, _dp(w), int(gnx), int(gny), C.c_double(hx),
                                            C.c_double(hy), C.c_int64(len(subdomains)), subs,
                                            _dp(packed), C.byref(sc), _dp(u),
                                            info.ctypes.data_as(C.c_void_p)), ctx.handle)
    out, off = [], 0
    for s, inf in zip(subdomains, info):
        n = s[2] * s[3]
        max_iters = cfg.max_iters if cfg.max_iters > 0 else 200 * max(s[2], s[3]) ** 2
        warn = "" if inf["converged"] else (
            f"Jacobi reached max_iters={max_iters} with update {inf['final_update']:.6f}")
        out.append(SolveResult(u[off:off + n].copy(), int(inf["iterations"]),
                               float(inf["final_update"]), bool(inf["converged"]), warn))
        off += n
    return out


def solve_dirichlet(w, nx, ny, hx, hy, bc: EdgeData, cfg: SolverConfig, ctx=None) -> SolveResult:
    """sdd::solve_dirichlet (proj/include/sdd/detsolver.hpp:44-45)."""
    w = _f64(w)
    if w.size != nx * ny:
        raise ValidationError("solve_dirichlet: weight array size mismatch")
    for a, n in zip(bc.arrays(), (nx, nx, ny, ny)):
        if len(a) != n:
            raise ValidationError("solve_dirichlet: boundary array sizes do not match grid")
    return solve_dirichlet_batch(w, nx, ny, hx, hy, [(0, 0, nx, ny)], [bc], cfg, ctx)[0]


# --------------------------------------------------------------- decomposition
@dataclass
class InterfaceLine:
    vertical: bool
    fixed_index: int
    fixed_coord: float
    length: int


@dataclass
class SubdomainLayout:
    """sdd::SubdomainLayout (decomposition.hpp:26-34)."""
    global_: GridSpec
    n_sub_x: int
    n_sub_y: int
    block_x: int
    block_y: int
    lines: list = field(default_factory=list)

    def subdomain(self, a, b):
        return (a * self.block_x, b * self.block_y, self.block_x + 1, self.block_y + 1)

    def subdomain_count(self):
        return self.n_sub_x * self.n_sub_y


def build_layout(spec: GridSpec, n_sub_x: int, n_sub_y: int) -> SubdomainLayout:
    """sdd::build_layout (proj/src/decomposition.cpp:26-53)."""
    if n_sub_x < 1 or n_sub_y < 1:
        raise LayoutError("build_layout: subdomain counts must be >= 1")
    if (spec.nx - 1) % n_sub_x:
        raise LayoutError(f"build_layout: nx-1={spec.nx - 1} not divisible by {n_sub_x} (x axis)")
    if (spec.ny - 1) % n_sub_y:
        raise LayoutError(f"build_layout: ny-1={spec.ny - 1} not divisible by {n_sub_y} (y axis)")
    lay = SubdomainLayout(spec, n_sub_x, n_sub_y, (spec.nx - 1) // n_sub_x, (spec.ny - 1) // n_sub_y)
    if lay.block_x < 2 or lay.block_y < 2:
        raise LayoutError("build_layout: subdomains need at least 3 nodes per axis")
    for a in range(1, n_sub_x):
        i = a * lay.block_x
        lay.lines.append(InterfaceLine(True, i, spec.node(i, 0)[0], spec.ny))
    for b in range(1, n_sub_y):
        j = b * lay.block_y
        lay.lines.append(InterfaceLine(False, j, spec.node(0, j)[1], spec.nx))
    return lay


@dataclass
class InterfacePlan:
    """sdd::InterfacePlan (decomposition.hpp:42-46)."""
    strategy: str
    k: int
    stochastic: list


def plan_interface_points(strategy: str, k: int, m: MonitorFunction,
                          layout: SubdomainLayout) -> InterfacePlan:
    """sdd::plan_interface_points (proj/src/decomposition.cpp:112-145)."""
    g = layout.global_
    cap = len(layout.lines) + 2
    nl = C.c_int32()
    vert, fixed, counts = (np.zeros(cap, np.int32) for _ in range(3))
    nodes = np.zeros(cap * max(g.nx, g.ny), np.int32)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
    d, dom = m.c(), g.domain.c()
    _check(lib().sddg_plan_interface_points(C.byref(d), C.byref(dom), g.nx, g.ny, layout.n_sub_x,
                                            layout.n_sub_y, PLACE.get(strategy, 99), int(k),
                                            C.byref(nl), ip(vert), ip(fixed), ip(counts), ip(nodes)))
    out, off = [], 0
    for l in range(nl.value):
        out.append(nodes[off:off + counts[l]].tolist())
        off += int(counts[l])
    return InterfacePlan(strategy, k, out)


@dataclass
class InterfaceSolution:
    """sdd::InterfaceSolution (decomposition.hpp:58-64)."""
    xi: list
    eta: list
    se_xi: list
    se_eta: list
    mc_points: int
    restarts: int
    warnings: int
    path_steps: int


def solve_interfaces(plan: InterfacePlan, m: MonitorFunction, bd: BoundaryData, cfg: WalkConfig,
                     layout: SubdomainLayout, ctx=None, interp: str = "linear") -> InterfaceSolution:
    """sdd::solve_interfaces (proj/include/sdd/decomposition.hpp:70-72).

    The plan must come from plan_interface_points on the same layout (the
    library re-derives it from (strategy, k))."""
    ctx = ctx or default_context()
    g = layout.global_
    lens = [ln.length for ln in layout.lines]
    tot = sum(lens)
    xi, eta, sx, se = (np.zeros(tot) for _ in range(4))
    st = _SddStats()
    d, dom, b, c = m.c(), g.domain.c(), bd.c(), cfg.c()
    o = SddOptions(interp=interp).c()
    _check(lib().sddg_solve_interfaces(ctx.handle, C.byref(d), C.byref(dom), g.nx, g.ny,
                                       layout.n_sub_x, layout.n_sub_y, PLACE.get(plan.strategy, 99),
                                       int(plan.k), C.byref(b), C.byref(c), C.byref(o), _dp(xi), _dp(eta),
                                       _dp(sx), _dp(se), C.byref(st)), ctx.handle)
    split = lambda a: [a[o:o + n].copy() for o, n in zip(np.cumsum([0] + lens[:-1]), lens)]
    return InterfaceSolution(split(xi), split(eta), split(sx), split(se), st.mc_points,
                             st.restarts, st.warnings, st.path_steps)


@dataclass
class SddResult:
    """sdd::SddResult (decomposition.hpp:79-86)."""
    xi: np.ndarray
    eta: np.ndarray
    t_stoc: float
    t_sub: float
    t_smooth: float
    mc_points: int
    subdomain_solves: int
    restarts: int
    path_steps: int
    warnings: int


class _SddOptions(C.Structure):
    _fields_ = [("smooth_interface", C.c_int32), ("smooth_span", C.c_int32), ("interp", C.c_int32),
                ("reserved", C.c_int32)]


@dataclass
class SddOptions:
    """sdd::SddOptions (proj/include/sdd/decomposition.hpp:74-77) + the
    interface fill ("linear" = reference, "spline" = BASELINE config 4)."""
    smooth_interface: bool = False
    smooth_span: int = 5
    interp: str = "linear"

    def c(self):
        return _SddOptions(1 if self.smooth_interface else 0, int(self.smooth_span),
                           INTERP.get(self.interp, 99), 0)


def solve_sdd(m: MonitorFunction, layout: SubdomainLayout, plan: InterfacePlan, wcfg: WalkConfig,
              scfg: SolverConfig, bc_mode=BC_REFERENCE, ctx=None,
              opts: SddOptions | None = None) -> SddResult:
    """sdd::solve_sdd (proj/include/sdd/decomposition.hpp:91-94)."""
    ctx = ctx or default_context()
    g = layout.global_
    xi, eta = np.zeros(g.nx * g.ny), np.zeros(g.nx * g.ny)
    st = _SddStats()
    d, dom, c, sc = m.c(), g.domain.c(), wcfg.c(), scfg.c()
    o = (opts or SddOptions()).c()
    _check(lib().sddg_solve_sdd(ctx.handle, C.byref(d), C.byref(dom), g.nx, g.ny, layout.n_sub_x,
                                layout.n_sub_y, PLACE.get(plan.strategy, 99), int(plan.k),
                                int(bc_mode), C.byref(c), C.byref(sc), C.byref(o), _dp(xi), _dp(eta),
                                C.byref(st)), ctx.handle)
    return SddResult(xi, eta, st.t_stoc, st.t_sub, st.t_smooth, st.mc_points, st.subdomain_solves,
                     st.restarts, st.path_steps, st.warnings)


# --------------------------------------------------------------- sharding seams
def interface_nodes(m: MonitorFunction, layout: SubdomainLayout, plan: InterfacePlan):
    """Unique Monte Carlo nodes of the plan in solve_interfaces order
    (sddg_interface_nodes): (px, py, point_id)."""
    g = layout.global_
    cap = max(1, sum(len(p) for p in plan.stochastic))
    px, py = np.zeros(cap), np.zeros(cap)
    pid = np.zeros(cap, np.uint64)
    n = C.c_int64()
    d, dom = m.c(), g.domain.c()
    _check(lib().sddg_interface_nodes(C.byref(d), C.byref(dom), g.nx, g.ny, layout.n_sub_x,
                                      layout.n_sub_y, PLACE.get(plan.strategy, 99), int(plan.k),
                                      C.c_int64(cap), _dp(px), _dp(py),
                                      pid.ctypes.data_as(C.c_void_p), C.byref(n)))
    k = n.value
    return px[:k].copy(), py[:k].copy(), pid[:k].copy()


def shard_plan(points, m: MonitorFunction, domain: RectDomain, cfg: WalkConfig, nranks: int):
    """sddg_shard_plan (host): (rank of each node, expected path-steps of each
    node's cfg.walks walks) -- the node shards of a multi-GPU context."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
    px, py = _f64(pts[:, 0]), _f64(pts[:, 1])
    rank = np.zeros(len(px), np.int32)
    cost = np.zeros(len(px))
    d, dom, c = m.c(), domain.c(), cfg.c()
    _check(lib().sddg_shard_plan(C.byref(d), C.byref(dom), C.byref(c), _dp(px), _dp(py),
                                 C.c_int64(len(px)), int(nranks), rank.ctypes.data_as(C.c_void_p),
                                 _dp(cost)))
    return rank, cost


def fill_interfaces(m: MonitorFunction, layout: SubdomainLayout, plan: InterfacePlan,
                    bd: BoundaryData, est: np.ndarray, interp: str = "linear") -> InterfaceSolution:
    """Interface lines from per-node estimates (sddg_fill_interfaces)."""
    g = layout.global_
    lens = [ln.length for ln in layout.lines]
    tot = sum(lens)
    xi, eta, sx, se = (np.zeros(tot) for _ in range(4))
    est = np.ascontiguousarray(est, dtype=ESTIMATE_DTYPE)
    d, dom, b = m.c(), g.domain.c(), bd.c()
    _check(lib().sddg_fill_interfaces(C.byref(d), C.byref(dom), g.nx, g.ny, layout.n_sub_x,
                                      layout.n_sub_y, PLACE.get(plan.strategy, 99), int(plan.k),
                                      C.byref(b), est.ctypes.data_as(C.c_void_p),
                                      C.c_int64(len(est)), C.byref(SddOptions(interp=interp).c()),
                                      _dp(xi), _dp(eta), _dp(sx), _dp(se)))
    split = lambda a: [a[o:o + n].copy() for o, n in zip(np.cumsum([0] + lens[:-1]), lens)]
    return InterfaceSolution(split(xi), split(eta), split(sx), split(se), len(est),
                             int(est["restarts"].sum()), int(est["warn"].sum()), 0)


def solve_subdomains(m: MonitorFunction, layout: SubdomainLayout, xi_lines, eta_lines,
                     scfg: SolverConfig, s_lo: int, s_hi: int, bc_mode=BC_REFERENCE, ctx=None):
    """Subdomain phase of solve_sdd for subdomains [s_lo, s_hi)
    (sddg_solve_subdomains): array (s_hi-s_lo, 2, ny_sub, nx_sub), field 0 = xi."""
    ctx = ctx or default_context()
    g = layout.global_
    bx, by = layout.block_x + 1, layout.block_y + 1
    ns = s_hi - s_lo
    fields = np.zeros(max(ns, 0) * 2 * bx * by)
    info = np.zeros(max(ns, 0) * 2, SOLVE_INFO_DTYPE)
    xl = _f64(np.concatenate(xi_lines)) if len(xi_lines) else np.zeros(0)
    el = _f64(np.concatenate(eta_lines)) if len(eta_lines) else np.zeros(0)
    d, dom, sc = m.c(), g.domain.c(), scfg.c()
    _check(lib().sddg_solve_subdomains(ctx.handle, C.byref(d), C.byref(dom), g.nx, g.ny,
                                       layout.n_sub_x, layout.n_sub_y, int(bc_mode), _dp(xl), _dp(el),
                                       C.byref(sc), int(s_lo), int(s_hi), _dp(fields),
                                       info.ctypes.data_as(C.c_void_p)), ctx.handle)
    return fields.reshape(ns, 2, by, bx), info


def assemble(layout: SubdomainLayout, fields: np.ndarray):
    """Global xi, eta from all subdomain blocks (solve_sdd assembly,
    proj/src/decomposition.cpp:357-377)."""
    g = layout.global_
    xi, eta = np.zeros((g.ny, g.nx)), np.zeros((g.ny, g.nx))
    for s in range(layout.subdomain_count()):
        i0, j0, nx, ny = layout.subdomain(s % layout.n_sub_x, s // layout.n_sub_x)
        xi[j0:j0 + ny, i0:i0 + nx] = fields[s, 0]
        eta[j0:j0 + ny, i0:i0 + nx] = fields[s, 1]
    return xi.ravel(), eta.ravel()


# --------------------------------------------------------------- post-processing
class _Quality(C.Structure):
    _fields_ = [("q_max", C.c_double), ("q_mean", C.c_double), ("r_max", C.c_double),
                ("r_mean", C.c_double), ("l_inf", C.c_double), ("has_reference", C.c_int32),
                ("has_l_inf", C.c_int32)]


@dataclass
class PhysicalMesh:
    """sdd::PhysicalMesh (field.hpp:36-51): x, y indexed b*m_xi + a."""
    m_xi: int
    m_eta: int
    domain: RectDomain
    x: np.ndarray
    y: np.ndarray


@dataclass
class QualityReport:
    """sdd::QualityReport (quality.hpp:10-14)."""
    q_max: float
    q_mean: float
    r_max: float | None = None
    r_mean: float | None = None
    l_inf: float | None = None


def invert_mesh(xi, eta, spec: GridSpec, m_xi: int, m_eta: int, ctx=None) -> PhysicalMesh:
    """sdd::invert_mesh (proj/include/sdd/invert.hpp:14) on the GPU."""
    ctx = ctx or default_context()
    xi, eta = _f64(xi), _f64(eta)
    if xi.size != spec.nx * spec.ny or eta.size != spec.nx * spec.ny:
        raise ValidationError("invert_mesh: field size does not match the grid")
    x, y = np.zeros(m_xi * m_eta), np.zeros(m_xi * m_eta)
    dom = spec.domain.c()
    _check(lib().sddg_invert_mesh(ctx.handle, _dp(xi), _dp(eta), spec.nx, spec.ny, C.byref(dom),
                                  int(m_xi), int(m_eta), _dp(x), _dp(y)), ctx.handle)
    return PhysicalMesh(m_xi, m_eta, spec.domain, x, y)


def quality_report(mesh: PhysicalMesh, reference: PhysicalMesh | None = None,
                   m: MonitorFunction | None = None, ctx=None) -> QualityReport:
    """sdd::quality_report (proj/src/quality.cpp:35-80) on the GPU."""
    ctx = ctx or default_context()
    if reference is not None and (reference.m_xi, reference.m_eta) != (mesh.m_xi, mesh.m_eta):
        raise ValidationError("quality_report: meshes have different node counts")
    q = _Quality()
    x, y = _f64(mesh.x), _f64(mesh.y)
    rx = _f64(reference.x) if reference is not None else None
    ry = _f64(reference.y) if reference is not None else None
    d = m.c() if (m is not None and reference is not None) else None
    _check(lib().sddg_quality_report(ctx.handle, _dp(x), _dp(y), mesh.m_xi, mesh.m_eta,
                                     _dp(rx) if rx is not None else None,
                                     _dp(ry) if ry is not None else None,
                                     C.byref(d) if d is not None else None, C.byref(q)), ctx.handle)
    return QualityReport(q.q_max, q.q_mean, q.r_max if q.has_reference else None,
                         q.r_mean if q.has_reference else None, q.l_inf if q.has_l_inf else None)


# --------------------------------------------------------------- smoothing
class _SmoothCfg(C.Structure):
    _fields_ = [("k", C.c_double), ("dt", C.c_double), ("steps", C.c_int32), ("scope", C.c_int32)]


@dataclass
class SmoothConfig:
    """sdd::SmoothConfig (proj/include/sdd/smoothing.hpp:15-22); scope
    "global" or "per_subdomain"."""
    k: float = 1000.0
    dt: float = 1e-4
    steps: int = 5
    scope: str = "global"


def perona_malik(xi, eta, spec: GridSpec, cfg: SmoothConfig, layout: SubdomainLayout | None = None,
                 ctx=None):
    """sdd::perona_malik (smoothing.hpp:34-35) on the GPU: returns (xi, eta,
    stability_warning)."""
    ctx = ctx or default_context()
    xi, eta = _f64(xi).copy(), _f64(eta).copy()
    scope = {"global": 0, "per_subdomain": 1}.get(cfg.scope, 99)
    if scope == 1 and layout is None:
        raise ValidationError("perona_malik: per-subdomain scope needs a layout")
    sx, sy = (layout.n_sub_x, layout.n_sub_y) if layout is not None else (1, 1)
    c = _SmoothCfg(cfg.k, cfg.dt, int(cfg.steps), scope)
    warn = C.c_int32()
    dom = spec.domain.c()
    _check(lib().sddg_perona_malik(ctx.handle, _dp(xi), _dp(eta), spec.nx, spec.ny, C.byref(dom),
                                   C.byref(c), sx, sy, C.byref(warn)), ctx.handle)
    return xi, eta, bool(warn.value)


def smooth_interface(values, span: int, ctx=None):
    """sdd::smooth_interface (smoothing.hpp:41) on the GPU."""
    ctx = ctx or default_context()
    v = _f64(values)
    out = np.zeros_like(v)
    _check(lib().sddg_smooth_interface(ctx.handle, _dp(v), len(v), int(span), _dp(out)), ctx.handle)
    return out


# --------------------------------------------------------------- stochastic-full, mesh IO
def stochastic_full(m: MonitorFunction, spec: GridSpec, cfg: WalkConfig, ctx=None):
    """The stochastic-full solve (run_stochastic_full, proj/src/cli.cpp:236-270):
    Monte Carlo at every interior node in one GPU batch.  Returns (xi, eta, stats)."""
    ctx = ctx or default_context()
    xi, eta = np.zeros(spec.nx * spec.ny), np.zeros(spec.nx * spec.ny)
    st = _SddStats()
    d, dom, c = m.c(), spec.domain.c(), cfg.c()
    _check(lib().sddg_stochastic_full(ctx.handle, C.byref(d), C.byref(dom), spec.nx, spec.ny,
                                      C.byref(c), _dp(xi), _dp(eta), C.byref(st)), ctx.handle)
    return xi, eta, {"t_stoc": st.t_stoc, "mc_points": st.mc_points, "restarts": st.restarts,
                     "path_steps": st.path_steps, "restart_warning": bool(st.warnings)}


def write_mesh(mesh: PhysicalMesh, xi, eta, spec: GridSpec, path: str):
    """sdd::write_mesh (proj/src/mesh_io.cpp:22-46): bit-exact sddmesh v1 text."""
    x, y, a, b = _f64(mesh.x), _f64(mesh.y), _f64(xi), _f64(eta)
    _check(lib().sddg_write_mesh(_dp(x), _dp(y), mesh.m_xi, mesh.m_eta, _dp(a), _dp(b), spec.nx,
                                 spec.ny, path.encode()))


def laplacian_smooth(xi, eta, spec: GridSpec, sweeps: int, ctx=None):
    """BASELINE config 4's "Laplacian smoothing, N sweeps" (sddg_laplacian_smooth):
    as the reference can express it, Perona-Malik FTCS with c = 1
    and dt = hx*hy/4, i.e. the 4-neighbour average for hx = hy; boundary kept."""
    ctx = ctx or default_context()
    xi2, eta2 = _f64(xi).copy(), _f64(eta).copy()
    if xi2.size != spec.nx * spec.ny or eta2.size != spec.nx * spec.ny:
        raise ValidationError("laplacian_smooth: field size does not match the grid")
    dom = spec.domain.c()
    _check(lib().sddg_laplacian_smooth(ctx.handle, _dp(xi2), _dp(eta2), spec.nx, spec.ny, C.byref(dom),
                                       int(sweeps)), ctx.handle)
    return xi2, eta2

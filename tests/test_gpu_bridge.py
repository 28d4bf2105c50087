"""The reference-side binding (integration/sddg_bridge.cpp)
compiled into the UNMODIFIED reference library: the linker's --wrap routes
the reference's own calls to sdd::mc_estimate and sdd::solve_dirichlet to
libsddg.so.  The reference's solve_interfaces (node dedupe, fill, crossing
reconciliation) and solve_sdd (boundary data, edge tables, assembly) then
consume GPU estimates and GPU subdomain solves, and must equal the
library's own sddg_solve_interfaces / sddg_solve_sdd bit for bit."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import bindings as B
from paper_1310_3435_b200 import sdd

pytestmark = pytest.mark.gpu
UNIT = sdd.RectDomain(0, 1, 0, 1)
ODOM = B.Domain(0, 1, 0, 1)
BRIDGE_SO = os.path.join(os.path.dirname(B.REF_SO), "libsddbridge.so")


@pytest.fixture(scope="module")
def bridge():
    if not os.path.exists(BRIDGE_SO):
        pytest.skip("oracle/_ref/libsddbridge.so not built (needs /root/reference)")
    sdd.lib()  # the same libsddg.so the bridge links
    br = B.Ref(path=BRIDGE_SO)
    br.L.sddg_bridge_configure.argtypes = [C.c_int, C.c_int, C.c_int]
    br.L.sddg_bridge_set_user_density.argtypes = [C.c_void_p]
    return br


def _use(br, m: sdd.MonitorFunction, on=True, method=sdd.JACOBI):
    br.L.sddg_bridge_configure(1 if on else 0, 0, method)
    d = m.c()
    br.L.sddg_bridge_set_user_density(C.addressof(d))
    br._keep = d


def test_reference_solve_interfaces_with_gpu_estimates(ctx, bridge):
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 65, 65)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("equispaced", 15, m, lay)
    bd = sdd.make_boundary_data(m, spec)
    mine = sdd.solve_interfaces(plan, m, bd, sdd.WalkConfig(scheme="linear", dt=1e-4, walks=2000, seed=1),
                                lay, ctx=ctx)
    _use(bridge, m)
    tabs = bridge.make_boundary(B.density(B.RING_W), ODOM, 65, 65)
    lines, mc, rs = bridge.solve_interfaces(B.density(B.RING_W), ODOM, 65, 65, 2, 2, 1, 15, tabs,
                                            B.walk_cfg(dt=1e-4, walks=2000, seed=1), threads=4)
    assert (mc, rs) == (mine.mc_points, mine.restarts)
    for l, (xi, eta, sxi, seta) in enumerate(lines):
        assert np.array_equal(xi, mine.xi[l]) and np.array_equal(eta, mine.eta[l])
        assert np.array_equal(sxi, mine.se_xi[l]) and np.array_equal(seta, mine.se_eta[l])


def test_reference_solve_sdd_with_gpu_walks_and_solves(ctx, bridge):
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 33, 33)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("equispaced", 7, m, lay)
    wcfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1000, seed=2)
    mine = sdd.solve_sdd(m, lay, plan, wcfg, sdd.SolverConfig(tol=1e-10, method="jacobi"), ctx=ctx)
    _use(bridge, m, method=sdd.JACOBI)
    xi, eta, _ = bridge.solve_sdd(B.density(B.RING_W), ODOM, 33, 33, 2, 2, 1, 7,
                                  B.walk_cfg(dt=1e-4, walks=1000, seed=2), tol=1e-10, threads=4)
    assert np.array_equal(xi, mine.xi) and np.array_equal(eta, mine.eta)
    # the reference's own CPU code through the same binary (bridge off): the
    # CUDA-vs-glibc libm differences stay below the 1e-10 bar
    _use(bridge, m, on=False)
    cxi, ceta, _ = bridge.solve_sdd(B.density(B.RING_W), ODOM, 33, 33, 2, 2, 1, 7,
                                    B.walk_cfg(dt=1e-4, walks=1000, seed=2), tol=1e-10, threads=0)
    assert np.max(np.abs(cxi - mine.xi)) <= 1e-10 and np.max(np.abs(ceta - mine.eta)) <= 1e-10


def test_any_user_density_through_a_table(ctx, bridge):
    # a user_supplied density the GPU knows nothing about, handed over as
    # samples (SDDG_DENS_TABLE); the reference sees user_supplied of the
    # same interpolant
    x = np.linspace(0, 1, 41)
    X, Y = np.meshgrid(x, x)
    rho = 1.0 + 3.0 * np.exp(-30.0 * ((X - 0.3) ** 2 + (Y - 0.6) ** 2)) + 0.5 * X * Y
    m = sdd.MonitorFunction.tabulated(rho, UNIT)
    spec = sdd.GridSpec(UNIT, 33, 33)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("optimal", 0, m, lay)
    wcfg = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=800, seed=4)
    mine = sdd.solve_sdd(m, lay, plan, wcfg, sdd.SolverConfig(tol=1e-10, method="jacobi"), ctx=ctx)
    _use(bridge, m)
    xi, eta, _ = bridge.solve_sdd(B.table_density(rho, ODOM), ODOM, 33, 33, 2, 2, 2, 0,
                                  B.walk_cfg(scheme="exp", lam=1000.0, walks=800, seed=4), tol=1e-10, threads=4)
    assert np.array_equal(xi, mine.xi) and np.array_equal(eta, mine.eta)

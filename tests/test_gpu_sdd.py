"""GPU end-to-end: solve_interfaces and solve_sdd through the C-ABI against
the reference's golden outputs and the reference test_decomposition.cpp
properties."""
import os
import subprocess

import numpy as np
import pytest

from oracle import bindings as B
from paper_1310_3435_b200 import sdd

pytestmark = pytest.mark.gpu
UNIT = sdd.RectDomain(0, 1, 0, 1)


def test_solve_interfaces_matches_reference(golden, ctx):
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 33, 33)
    bd = sdd.make_boundary_data(m, spec)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("equispaced", 5, m, lay)
    s = sdd.solve_interfaces(plan, m, bd, sdd.WalkConfig(scheme="linear", dt=1e-4, walks=200, seed=1),
                             lay, ctx=ctx)
    want = golden["ifc_ring33"]
    got = [np.concatenate(v) for v in (s.xi, s.eta, s.se_xi, s.se_eta)]
    for k in range(4):
        assert np.max(np.abs(got[k] - want[k])) <= 1e-10
    assert (s.mc_points, s.restarts) == tuple(int(v) for v in golden["ifc_ring33_meta"])


def test_solve_sdd_matches_reference(golden, ctx):
    m = sdd.MonitorFunction.running_example()
    spec = sdd.GridSpec(UNIT, 33, 33)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("equispaced", 5, m, lay)
    r = sdd.solve_sdd(m, lay, plan, sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=200, seed=1),
                      sdd.SolverConfig(tol=1e-12), ctx=ctx)
    assert np.max(np.abs(r.xi - golden["sdd_running33_xi"])) <= 1e-10
    assert np.max(np.abs(r.eta - golden["sdd_running33_eta"])) <= 1e-10
    assert r.subdomain_solves == 8 and r.mc_points > 0 and r.path_steps > 0


def test_one_by_one_layout_is_the_single_domain_solve(oracle, ctx):
    # proj/tests/test_decomposition.cpp:164-179
    m = sdd.MonitorFunction.running_example()
    spec = sdd.GridSpec(UNIT, 29, 29)
    lay = sdd.build_layout(spec, 1, 1)
    plan = sdd.plan_interface_points("all", 0, m, lay)
    r = sdd.solve_sdd(m, lay, plan, sdd.WalkConfig(walks=10, seed=1), sdd.SolverConfig(tol=1e-10), ctx=ctx)
    odom = B.Domain(0, 1, 0, 1)
    w = oracle.weight_values(B.density(B.RUNNING), odom, 29, 29)
    t = oracle.make_boundary(B.density(B.RUNNING), odom, 29, 29)
    u_xi, *_ = oracle.solve_dirichlet(w, 29, 29, 1 / 28, 1 / 28, *t.f, tol=1e-10)
    u_eta, *_ = oracle.solve_dirichlet(w, 29, 29, 1 / 28, 1 / 28, *t.g, tol=1e-10)
    assert np.array_equal(r.xi, u_xi) and np.array_equal(r.eta, u_eta)
    assert r.mc_points == 0


def test_uniform_weight_interface_is_xi_equals_x(ctx):
    # proj/tests/test_decomposition.cpp:119-138
    m = sdd.MonitorFunction.constant()
    spec = sdd.GridSpec(UNIT, 17, 17)
    lay = sdd.build_layout(spec, 2, 2)
    bd = sdd.make_boundary_data(m, spec)
    plan = sdd.plan_interface_points("all", 0, m, lay)
    s = sdd.solve_interfaces(plan, m, bd, sdd.WalkConfig(scheme="exponential", lambda_=2000, walks=2000, seed=1),
                             lay, ctx=ctx)
    assert len(s.xi) == 2
    for pos in range(1, 16):
        assert abs(s.xi[0][pos] - 0.5) <= 4.0 * s.se_xi[0][pos] + 1e-6
    assert s.xi[0][0] == bd.f.bottom[8] and s.xi[0][16] == bd.f.top[8]
    assert s.eta[0][0] == 0.0 and s.eta[0][16] == 1.0
    assert s.mc_points == 2 * 15 - 1


def test_solve_sdd_deterministic(ctx):
    # proj/tests/test_decomposition.cpp:181-195 (thread counts -> repeated launches)
    m = sdd.MonitorFunction.running_example()
    lay = sdd.build_layout(sdd.GridSpec(UNIT, 17, 17), 2, 2)
    plan = sdd.plan_interface_points("optimal", 0, m, lay)
    cfg = sdd.WalkConfig(scheme="exponential", lambda_=1000, walks=1500, seed=9)
    a = sdd.solve_sdd(m, lay, plan, cfg, sdd.SolverConfig(), ctx=ctx)
    b = sdd.solve_sdd(m, lay, plan, cfg, sdd.SolverConfig(), ctx=ctx)
    assert np.array_equal(a.xi, b.xi) and np.array_equal(a.eta, b.eta)


def test_interface_values_carried_into_subdomain_edges(ctx):
    # proj/tests/test_decomposition.cpp:197-218: the assembled mesh carries
    # the interface line values unchanged
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 33, 33)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("equispaced", 7, m, lay)
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=300, seed=3)
    r = sdd.solve_sdd(m, lay, plan, cfg, sdd.SolverConfig(tol=1e-12, method="rbsor"), ctx=ctx)
    s = sdd.solve_interfaces(plan, m, sdd.make_boundary_data(m, spec), cfg, lay, ctx=ctx)
    X = r.xi.reshape(33, 33)
    assert np.array_equal(X[:, 16], s.xi[0])   # vertical line i = 16
    assert np.array_equal(X[16, :], s.xi[1])   # horizontal line j = 16


def test_sdd_close_to_single_domain(oracle, ctx):
    # proj/tests/test_decomposition.cpp:140-162: uniform weight, within 0.02
    m = sdd.MonitorFunction.constant()
    spec = sdd.GridSpec(UNIT, 17, 17)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("all", 0, m, lay)
    r = sdd.solve_sdd(m, lay, plan, sdd.WalkConfig(scheme="exponential", lambda_=2000, walks=2000, seed=1),
                      sdd.SolverConfig(), ctx=ctx)
    assert r.subdomain_solves == 8 and r.mc_points == 29
    odom = B.Domain(0, 1, 0, 1)
    w = oracle.weight_values(B.density(B.CONSTANT), odom, 17, 17)
    t = oracle.make_boundary(B.density(B.CONSTANT), odom, 17, 17)
    u_xi, *_ = oracle.solve_dirichlet(w, 17, 17, 1 / 16, 1 / 16, *t.f)
    u_eta, *_ = oracle.solve_dirichlet(w, 17, 17, 1 / 16, 1 / 16, *t.g)
    assert max(np.max(np.abs(r.xi - u_xi)), np.max(np.abs(r.eta - u_eta))) <= 0.02


def test_identity_bc_mode(ctx):
    m = sdd.MonitorFunction.ring(analytic=True)
    spec = sdd.GridSpec(UNIT, 65, 65)
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("equispaced", 31, m, lay)
    r = sdd.solve_sdd(m, lay, plan, sdd.WalkConfig(scheme="linear", dt=1e-4, walks=500, seed=1),
                      sdd.SolverConfig(tol=1e-10, method="rbsor"), bc_mode=sdd.BC_IDENTITY, ctx=ctx)
    X = r.xi.reshape(65, 65)
    assert np.allclose(X[0, :], np.arange(65) / 64, atol=1e-15)
    assert (X >= 0).all() and (X <= 1).all()


def test_distributed_solve_sdd_world1_matches_solve_sdd(ctx):
    # the sharded driver (paper_1310_3435_b200.parallel) over NCCL at world
    # size 1 reproduces solve_sdd bit for bit
    import socket
    import torch
    import torch.distributed as dist
    from paper_1310_3435_b200 import parallel
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    try:
        m = sdd.MonitorFunction.ring(analytic=True)
        lay = sdd.build_layout(sdd.GridSpec(UNIT, 65, 65), 4, 4)
        plan = sdd.plan_interface_points("all", 0, m, lay)
        wcfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=400, seed=3)
        scfg = sdd.SolverConfig(tol=1e-11, method="rbsor")
        xi, eta, ifc, est = parallel.solve_sdd_distributed(m, lay, plan, wcfg, scfg, ctx=ctx)
        r = sdd.solve_sdd(m, lay, plan, wcfg, scfg, ctx=ctx)
        assert np.array_equal(xi, r.xi) and np.array_equal(eta, r.eta)
        assert len(est) == r.mc_points
    finally:
        dist.destroy_process_group()


def test_stochastic_full_matches_reference_estimates(ctx, oracle):
    # run_stochastic_full (proj/src/cli.cpp:236-270): every interior node
    m = sdd.MonitorFunction.running_example()
    spec = sdd.GridSpec(UNIT, 9, 9)
    cfg = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=300, seed=5)
    xi, eta, st = sdd.stochastic_full(m, spec, cfg, ctx=ctx)
    assert st["mc_points"] == 49 and not st["restart_warning"]
    odom = B.Domain(0, 1, 0, 1)
    t = oracle.make_boundary(B.density(B.RUNNING), odom, 9, 9)
    pts = [(i / 8, j / 8) for j in range(1, 8) for i in range(1, 8)]
    pid = [j * 9 + i for j in range(1, 8) for i in range(1, 8)]
    o = oracle.mc_estimate_batch(B.density(B.RUNNING), odom, t, B.walk_cfg(scheme="exp", lam=1000.0, walks=300, seed=5),
                                 [p[0] for p in pts], [p[1] for p in pts], pid, threads=8)
    assert np.max(np.abs(xi[pid] - o["xi"])) <= 1e-10 and np.max(np.abs(eta[pid] - o["eta"])) <= 1e-10
    assert np.array_equal(xi.reshape(9, 9)[0], t.f[0]) and np.array_equal(eta.reshape(9, 9)[:, 0], t.g[2])


@pytest.mark.parametrize("mode", ["reference", "analytic"])
def test_plain_c_caller_matches_python_mirror(ctx, mode):
    # examples/sdd_config1.c runs BASELINE config 1 end to end through the
    # C-ABI alone; the Python mirror's solve_sdd on the same inputs gives the
    # same mesh bit for bit (checksums in index order) and the same counts
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([os.path.join(root, "examples", "_bin", "sdd_config1"), mode, "1"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    mc, steps, _, _, sx, se, qmax, qmean = out.stdout.split()
    m = sdd.MonitorFunction.ring(analytic=mode == "analytic")
    spec = sdd.GridSpec(UNIT, 65, 65)
    lay = sdd.build_layout(spec, 2, 2)
    r = sdd.solve_sdd(m, lay, sdd.plan_interface_points("equispaced", 31, m, lay),
                      sdd.WalkConfig(scheme="linear", dt=1e-4, walks=10_000, seed=1),
                      sdd.SolverConfig(tol=1e-10, method="rbsor"), ctx=ctx)
    assert int(mc) == r.mc_points == 61 and int(steps) == r.path_steps
    # the C program sums in index order (np.cumsum is sequential; np.sum is pairwise)
    assert float(sx) == float(np.cumsum(r.xi)[-1]) and float(se) == float(np.cumsum(r.eta)[-1])
    q = sdd.quality_report(sdd.invert_mesh(r.xi, r.eta, spec, 65, 65, ctx=ctx), ctx=ctx)
    assert float(qmax) == q.q_max and float(qmean) == q.q_mean


def test_plain_c_caller_on_a_multi_gpu_context():
    # the same C program through sddg_create_multi: device 0 listed three
    # times (three ranks: sharded nodes and subdomains, device-copy exchange)
    # prints the single-device mesh checksums bit for bit
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "examples", "_bin", "sdd_config1")
    one = subprocess.run([exe, "analytic", "3"], capture_output=True, text=True, timeout=300)
    three = subprocess.run([exe, "analytic", "3", "0,0,0"], capture_output=True, text=True, timeout=300)
    assert one.returncode == 0 and three.returncode == 0, (one.stderr, three.stderr)
    a, b = one.stdout.split(), three.stdout.split()
    assert a[:2] == b[:2] and a[4:] == b[4:]  # all but the two timings

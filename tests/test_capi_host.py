"""CPU-side checks of the C-ABI library (no compute calls need a GPU here).

* libsddg.so loads and exports every function declared in include/sddg.h;
* the host-side set-up entry points (boundary tables, layout + placement)
  reproduce the reference's golden outputs bit for bit;
* errors map onto the reference's exception classes;
* without a GPU, creating a context fails loudly (no CPU fallback).
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from cases import plan_from_flat
from oracle import bindings as B
from paper_1310_3435_b200 import sdd

UNIT = sdd.RectDomain(0, 1, 0, 1)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "sddg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sddg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 15
    lib = sdd.lib()
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", sdd.library_path()], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (sddg_\w+)", out))
    assert set(names) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", sdd.library_path()], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_abi_version():
    assert sdd.lib().sddg_abi_version() == 2
    assert b"sm_100a" in sdd.lib().sddg_version()


@pytest.mark.parametrize("key,kind,dom", [
    ("ring_65", sdd.RING_W, (0, 1, 0, 1)), ("shock_129", sdd.SHOCK_W, (0, 1, 0, 1)),
    ("twobump_33", sdd.TWOBUMP_W, (0, 1, 0, 1)), ("running_29", sdd.RUNNING, (0, 1, 0, 1)),
    ("five_ring_17", sdd.FIVE_RING, (-1, 1, -1, 1)), ("constant_33", sdd.CONSTANT, (0, 1, 0, 1)),
    ("huang_sloan_33", sdd.HUANG_SLOAN, (0, 1, 0, 1)), ("mackenzie_33", sdd.MACKENZIE, (0, 1, 0, 1))])
def test_make_boundary_data_matches_reference(golden, key, kind, dom):
    n = int(key.rsplit("_", 1)[1])
    m = {sdd.CONSTANT: sdd.MonitorFunction.constant(), sdd.RUNNING: sdd.MonitorFunction.running_example(),
         sdd.HUANG_SLOAN: sdd.MonitorFunction.huang_sloan(), sdd.MACKENZIE: sdd.MonitorFunction.mackenzie(),
         sdd.FIVE_RING: sdd.MonitorFunction.five_ring()}.get(kind) or sdd.MonitorFunction.weight(kind)
    bd = sdd.make_boundary_data(m, sdd.GridSpec(sdd.RectDomain(*dom), n, n))
    got = np.concatenate(bd.f.arrays() + bd.g.arrays())
    assert np.array_equal(got, golden[f"tables_{key}"])


def test_identity_boundary_tables():
    bd = sdd.make_boundary_data(sdd.MonitorFunction.ring(), sdd.GridSpec(sdd.RectDomain(0, 1, 0, 1), 65, 65),
                                mode=sdd.BC_IDENTITY)
    x = np.arange(65) / 64
    assert np.allclose(bd.f.bottom, x, atol=1e-15) and np.allclose(bd.g.left, x, atol=1e-15)
    assert (bd.f.left == 0).all() and (bd.f.right == 1).all()


@pytest.mark.parametrize("name,m,n,sx,strategy,k", [
    ("running29_all", sdd.MonitorFunction.running_example(), 29, 2, "all", 0),
    ("running29_eq7", sdd.MonitorFunction.running_example(), 29, 2, "equispaced", 7),
    ("running29_opt", sdd.MonitorFunction.running_example(), 29, 2, "optimal", 0),
    ("constant29_opt", sdd.MonitorFunction.constant(), 29, 2, "optimal", 0),
    ("ring65_eq31", sdd.MonitorFunction.ring(), 65, 2, "equispaced", 31),
    ("twobump513_opt", sdd.MonitorFunction.two_bump(), 513, 4, "optimal", 0),
    ("five157_opt", sdd.MonitorFunction.five_ring(), 157, 4, "optimal", 0),
    ("shock129_eq40", sdd.MonitorFunction.shock(), 129, 4, "equispaced", 40)])
def test_plans_match_reference(golden, name, m, n, sx, strategy, k):
    spec = sdd.GridSpec(m.domain, n, n)
    lay = sdd.build_layout(spec, sx, sx)
    plan = sdd.plan_interface_points(strategy, k, m, lay)
    want = plan_from_flat(golden[f"plan_{name}"])
    assert [(ln.vertical, ln.fixed_index) for ln in lay.lines] == [(v, f) for v, f, _ in want]
    assert plan.stochastic == [nodes for _, _, nodes in want]


def test_layout_arithmetic():
    # proj/tests/test_decomposition.cpp:28-62
    unit = sdd.RectDomain(0, 1, 0, 1)
    lay = sdd.build_layout(sdd.GridSpec(unit, 29, 29), 2, 2)
    assert (lay.block_x, lay.block_y, len(lay.lines)) == (14, 14, 2)
    assert lay.lines[0].vertical and not lay.lines[1].vertical
    assert lay.subdomain(1, 0) == (14, 0, 15, 15)
    lay = sdd.build_layout(sdd.GridSpec(unit, 157, 157), 4, 4)
    assert lay.subdomain_count() == 16 and lay.block_x == 39 and len(lay.lines) == 6
    assert sdd.build_layout(sdd.GridSpec(unit, 29, 29), 1, 1).lines == []
    with pytest.raises(sdd.LayoutError, match="x axis"):
        sdd.build_layout(sdd.GridSpec(unit, 29, 29), 3, 2)
    with pytest.raises(sdd.LayoutError, match="y axis"):
        sdd.build_layout(sdd.GridSpec(unit, 29, 29), 2, 5)


def test_validation_errors_on_host_entry_points():
    m = sdd.MonitorFunction.running_example()
    lay = sdd.build_layout(sdd.GridSpec(sdd.RectDomain(0, 1, 0, 1), 29, 29), 2, 2)
    with pytest.raises(sdd.ValidationError):
        sdd.plan_interface_points("equispaced", 0, m, lay)
    with pytest.raises(sdd.ValidationError):
        sdd.plan_interface_points("equispaced", 28, m, lay)
    with pytest.raises(sdd.ValidationError):
        sdd.GridSpec(sdd.RectDomain(0, 1, 0, 1), 2, 5)
    with pytest.raises(sdd.ValidationError):
        sdd.RectDomain(1, 0, 0, 1)


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(sdd.CudaError):
        sdd.Context(0)


def test_write_mesh_is_byte_identical_to_reference(golden, tmp_path, refimpl):
    # sddmesh v1 (proj/src/mesh_io.cpp:22-46): same bytes as the reference writer
    X = golden["invert_sdd_running33"]
    xi, eta = golden["sdd_running33_xi"], golden["sdd_running33_eta"]
    spec = sdd.GridSpec(sdd.RectDomain(0, 1, 0, 1), 33, 33)
    mesh = sdd.PhysicalMesh(33, 33, spec.domain, X[0], X[1])
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    sdd.write_mesh(mesh, xi, eta, spec, str(ours))
    refimpl.write_mesh(X[0], X[1], 33, 33, xi, eta, 33, 33, str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
    assert ours.read_bytes().startswith(b"sddmesh v1 33 33\n")
    with pytest.raises(sdd.ValidationError):
        sdd.write_mesh(mesh, xi, eta, sdd.GridSpec(spec.domain, 33, 17), str(ours))


def test_plain_c_caller_builds_links_and_fails_loudly_without_a_gpu():
    # examples/sdd_config1.c: a C99 program against include/sddg.h only,
    # built by build() and linked to the in-tree library; with no usable GPU
    # the first call reports SDDG_ERR_CUDA (status 6) -- no CPU fallback
    exe = os.path.join(ROOT, "examples", "_bin", "sdd_config1")
    if not os.path.exists(exe):
        from paper_1310_3435_b200 import build as bld
        bld.build()
    ldd = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "paper_1310_3435_b200/_lib/libsddg.so" in ldd
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present: tests/test_gpu_sdd.py runs the program")
    except ImportError:
        pass
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and "status 6" in r.stderr


def test_shard_plan_exit_time_model_known_answer():
    # the cost model behind the multi-GPU node shards: expected first-exit
    # time T of dX = grad(w)/w dt + sqrt(2) dW, div(w grad T) = -w, T = 0 on
    # the edges.  Constant w on the unit square: T solves Laplace(T) = -1,
    # whose centre value is the square's torsion constant 0.0736713...
    m = sdd.MonitorFunction.constant()
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=10)
    rank, cost = sdd.shard_plan([(0.5, 0.5), (0.25, 0.5), (0.05, 0.05)], m, UNIT, cfg, 2)
    t_centre = (cost[0] / 10 - 1) * 1e-4
    assert abs(t_centre - 0.0736713) < 2e-4
    assert cost[0] > cost[1] > cost[2]
    assert rank.tolist() == [0, 1, 1]          # LPT: the largest alone, the rest on the other rank
    # exponential scheme: mean step 1/lambda
    _, ce = sdd.shard_plan([(0.5, 0.5)], m, UNIT, sdd.WalkConfig(scheme="exponential", lambda_=1000.0,
                                                                  walks=1), 1)
    assert abs((ce[0] - 1) / 1000 - t_centre) < 1e-9


def test_shard_plan_tracks_the_density():
    # a strong monitor (shock layer, w up to 21) slows walks down where w is
    # large only through the drift; the plan must be deterministic, cover
    # every node once and be balanced
    m = sdd.MonitorFunction.shock()
    rng = np.random.default_rng(2)
    pts = rng.uniform(0.02, 0.98, (3000, 2))
    cfg = sdd.WalkConfig(scheme="linear", dt=1e-5, walks=1000)
    r1, c1 = sdd.shard_plan(pts, m, UNIT, cfg, 8)
    r2, c2 = sdd.shard_plan(pts, m, UNIT, cfg, 8)
    assert np.array_equal(r1, r2) and np.array_equal(c1, c2)
    loads = np.array([c1[r1 == r].sum() for r in range(8)])
    assert loads.max() / loads.min() < 1.001
    with pytest.raises(sdd.OutOfDomainError):
        sdd.shard_plan([(0.0, 0.5)], m, UNIT, cfg, 2)
    with pytest.raises(sdd.ValidationError):
        sdd.shard_plan(pts, m, UNIT, cfg, 0)


def test_nccl_loaded_at_run_time_and_torch_still_imports():
    # libsddg links no NCCL; the first multi-GPU call loads one at run time,
    # and it must be the copy PyTorch links (a second libnccl.so.2 loaded
    # first would shadow torch's), so torch imports fine afterwards
    import sys
    code = ("from paper_1310_3435_b200 import sdd; i = sdd.nccl_unique_id(); assert len(i) == 128; "
            "import torch, torch.distributed; "
            "maps = open('/proc/self/maps').read(); "
            "libs = {l.split()[-1] for l in maps.splitlines() if 'libnccl' in l}; "
            "assert len(libs) == 1, libs; print(libs.pop())")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    out = subprocess.run(["readelf", "-d", sdd.library_path()], capture_output=True, text=True).stdout
    assert "nccl" not in out

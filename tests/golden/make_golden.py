"""Generate tests/golden/golden.npz from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libsddref.so, compiled by
oracle/Makefile from /root/reference/proj/src) through its public API and
stores small input/output vectors: Philox blocks, stream words and normals,
densities and drifts, boundary tables, per-path walk results (run_walk replay),
mc_estimate records, solve_dirichlet fields, interface plans, solve_interfaces
lines and a solve_sdd mesh.  The reference has no golden vectors of its own
(SURVEY.md 8(c)), so these pin both the C restatement (oracle/sdd_oracle.c)
and the GPU kernels.

    make -C oracle ref && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import bindings as B  # noqa: E402

OUT = os.path.join(HERE, "golden.npz")
UNIT = B.Domain(0, 1, 0, 1)
FIVE = B.Domain(-1, 1, -1, 1)

# (name, kind, domain)
DENSITIES = [("constant", B.CONSTANT, UNIT), ("running", B.RUNNING, UNIT),
             ("huang_sloan", B.HUANG_SLOAN, UNIT), ("mackenzie", B.MACKENZIE, UNIT),
             ("five_ring", B.FIVE_RING, FIVE), ("ring", B.RING_W, UNIT),
             ("shock", B.SHOCK_W, UNIT), ("twobump", B.TWOBUMP_W, UNIT)]

# walk dump cases: name, density, grid n, scheme cfg kwargs, start, point_id, n walks
DUMPS = [
    ("ring_lin_center", B.RING_W, 65, dict(dt=1e-4, seed=1), (0.5, 0.5), 32 * 65 + 32, 128),
    ("ring_lin_edge", B.RING_W, 65, dict(dt=1e-4, seed=1), (0.5, 2 / 64), 2 * 65 + 32, 128),
    ("ring_lin_nobridge", B.RING_W, 65, dict(dt=1e-4, seed=2, bridge=False), (0.5, 0.5), 2112, 64),
    ("shock_lin", B.SHOCK_W, 129, dict(dt=1e-4, seed=1), (0.5, 0.5), 64 * 129 + 64, 64),
    ("twobump_lin", B.TWOBUMP_W, 33, dict(dt=1e-4, seed=4), (0.3, 0.3), 123, 64),
    ("running_exp", B.RUNNING, 17, dict(scheme="exp", lam=1000.0, seed=3), (0.3, 0.6), 99, 128),
    ("five_ring_exp", B.FIVE_RING, 33, dict(scheme="exp", lam=1000.0, seed=5), (0.1, -0.2), 7, 64),
    ("constant_restart", B.CONSTANT, 33, dict(dt=1e-4, seed=7, max_steps=300), (0.02, 0.5), 1, 128),
    ("huang_lin_bigpid", B.HUANG_SLOAN, 33, dict(dt=1e-3, seed=(1 << 40) + 9), (0.7, 0.4),
     (1 << 45) + 12345, 64),
    ("mackenzie_lin", B.MACKENZIE, 33, dict(dt=1e-3, seed=11), (0.4, 0.45), 5, 64),
]

# estimate cases: name, density, grid, cfg kwargs, points, pids
ESTIMATES = [
    ("ring_1000", B.RING_W, 65, dict(dt=1e-4, seed=1, walks=1000),
     [(0.5, 0.5), (0.5, 2 / 64), (16 / 64, 0.5)], [2112, 162, 32 * 65 + 16]),
    ("running_exp_300", B.RUNNING, 17, dict(scheme="exp", lam=1000.0, seed=42, walks=300),
     [(0.3, 0.6), (0.75, 0.5)], [99, 100]),
    ("constant_walks1", B.CONSTANT, 33, dict(dt=1e-4, seed=1, walks=1), [(0.5, 0.5)], [0]),
    ("constant_restart", B.CONSTANT, 33, dict(dt=1e-4, seed=7, walks=400, max_steps=3),
     [(0.02, 0.5)], [1]),
]


def main():
    ref = B.Ref()
    G = {}
    rng = np.random.default_rng(20241020)
    # -- Philox blocks (rng.hpp:12-29)
    keys = [(0, 0), (1, 0), (0xFFFFFFFF, 0xFFFFFFFF), (123456789, 987654321)]
    ctrs = [(0, 0, 0, 0), (1, 2, 3, 4), (0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF),
            (7, 3, 2112, (5 << 16) | 0x1234)]
    kc = np.array([[k[0], k[1], *c] for k in keys for c in ctrs], np.uint64)
    G["philox_in"] = kc
    G["philox_out"] = np.array([ref.philox_block(int(r[0]), int(r[1]), [int(v) for v in r[2:]])
                                for r in kc], np.uint64)
    # -- streams (rng.hpp:31-83)
    streams = np.array([(1, 7, 3, 0), (2, 7, 3, 0), (1, 8, 3, 0), (1, 7, 4, 0), (1, 7, 3, 5),
                        ((1 << 40) + 3, (1 << 47) + 5, 4000000000, 1023), (0, 0, 0, 0)], np.uint64)
    G["stream_keys"] = streams
    G["stream_u64"] = np.stack([ref.stream_u64(*[int(v) for v in s], 64) for s in streams])
    G["stream_u01"] = np.stack([ref.stream_u01(*[int(v) for v in s], 32) for s in streams])
    G["stream_u01_open"] = np.stack([ref.stream_u01(*[int(v) for v in s], 32, True) for s in streams])
    G["stream_normals"] = np.stack([ref.stream_normals(*[int(v) for v in s], 32) for s in streams])
    # -- densities and drifts (monitor.cpp:121-240)
    for name, kind, dom in DENSITIES:
        x = dom.xmin + (dom.xmax - dom.xmin) * (0.01 + 0.98 * rng.random(64))
        y = dom.ymin + (dom.ymax - dom.ymin) * (0.01 + 0.98 * rng.random(64))
        rho, bx, by = ref.rho_drift(B.density(kind), dom, x, y)
        G[f"dens_{name}_xy"] = np.stack([x, y])
        G[f"dens_{name}_out"] = np.stack([rho, bx, by])
    # -- boundary tables (boundary.cpp:44-56)
    for name, kind, dom, n in [("ring", B.RING_W, UNIT, 65), ("shock", B.SHOCK_W, UNIT, 129),
                               ("twobump", B.TWOBUMP_W, UNIT, 33), ("running", B.RUNNING, UNIT, 29),
                               ("five_ring", B.FIVE_RING, FIVE, 17), ("five_ring", B.FIVE_RING, FIVE, 33),
                               ("constant", B.CONSTANT, UNIT, 33),
                               ("huang_sloan", B.HUANG_SLOAN, UNIT, 33),
                               ("mackenzie", B.MACKENZIE, UNIT, 33), ("running17", B.RUNNING, UNIT, 17)]:
        t = ref.make_boundary(B.density(kind), dom, n, n)
        G[f"tables_{name}_{n}"] = np.concatenate(t.f + t.g)
    # -- walk dumps (run_walk replay, sde.cpp:151-183)
    for name, kind, n, kw, p, pid, nw in DUMPS:
        dom = FIVE if kind == B.FIVE_RING else UNIT
        t = ref.make_boundary(B.density(kind), dom, n, n)
        cfg = B.walk_cfg(**kw)
        d = ref.walk_dump(B.density(kind), dom, t, cfg, p[0], p[1], pid, 0, nw)
        G[f"dump_{name}"] = d.view(np.uint8)
    # -- estimates (mc_estimate, sde.cpp:193-246)
    for name, kind, n, kw, pts, pids in ESTIMATES:
        t = ref.make_boundary(B.density(kind), UNIT, n, n)
        cfg = B.walk_cfg(**kw)
        e = ref.mc_estimate_batch(B.density(kind), UNIT, t, cfg, [p[0] for p in pts],
                                  [p[1] for p in pts], pids, threads=4)
        G[f"est_{name}"] = e.view(np.uint8)
    # -- solve_dirichlet (detsolver.cpp:72-209)
    solves = [("ring17_t10", B.RING_W, 17, 17, 1e-10, 0, True),
              ("running33x17_t8", B.RUNNING, 33, 17, 1e-8, 0, True),
              ("twobump17_noblend", B.TWOBUMP_W, 17, 17, 1e-9, 0, False),
              ("ring33_maxit", B.RING_W, 33, 33, 1e-12, 50, True),
              ("shock33_t13", B.SHOCK_W, 33, 33, 1e-13, 0, True)]
    for name, kind, nx, ny, tol, mi, blend in solves:
        w = ref.weight_values(B.density(kind), UNIT, nx, ny)
        t = ref.make_boundary(B.density(kind), UNIT, nx, ny)
        for fld, tabs in (("xi", t.f), ("eta", t.g)):
            u, it, fu, cv = ref.solve_dirichlet(w, nx, ny, 1.0 / (nx - 1), 1.0 / (ny - 1), *tabs,
                                                tol=tol, max_iters=mi, init_blend=blend)
            G[f"solve_{name}_{fld}_u"] = u
            G[f"solve_{name}_{fld}_info"] = np.array([it, fu, cv], np.float64)
        G[f"solve_{name}_w"] = w
    # -- plans (decomposition.cpp:112-145)
    plans = [("running29_all", B.RUNNING, UNIT, 29, 2, 2, 0, 0),
             ("running29_eq7", B.RUNNING, UNIT, 29, 2, 2, 1, 7),
             ("running29_opt", B.RUNNING, UNIT, 29, 2, 2, 2, 0),
             ("constant29_opt", B.CONSTANT, UNIT, 29, 2, 2, 2, 0),
             ("ring65_eq31", B.RING_W, UNIT, 65, 2, 2, 1, 31),
             ("twobump513_opt", B.TWOBUMP_W, UNIT, 513, 4, 4, 2, 0),
             ("five157_opt", B.FIVE_RING, FIVE, 157, 4, 4, 2, 0),
             ("shock129_eq40", B.SHOCK_W, UNIT, 129, 4, 4, 1, 40)]
    for name, kind, dom, n, sx, sy, st, k in plans:
        lines = ref.plan(B.density(kind), dom, n, n, sx, sy, st, k)
        flat = []
        for v, fi, nodes in lines:
            flat += [int(v), fi, len(nodes)] + list(nodes)
        G[f"plan_{name}"] = np.array(flat, np.int64)
    # -- solve_interfaces and solve_sdd (decomposition.cpp:147-385)
    t = ref.make_boundary(B.density(B.RING_W), UNIT, 33, 33)
    lines, mc, rs = ref.solve_interfaces(B.density(B.RING_W), UNIT, 33, 33, 2, 2, 1, 5, t,
                                         B.walk_cfg(dt=1e-4, seed=1, walks=200), threads=4)
    G["ifc_ring33"] = np.stack([np.concatenate([l[k] for l in lines]) for k in range(4)])
    G["ifc_ring33_meta"] = np.array([mc, rs])
    xi, eta, _ = ref.solve_sdd(B.density(B.RUNNING), UNIT, 33, 33, 2, 2, 1, 5,
                               B.walk_cfg(scheme="exp", lam=1000.0, seed=1, walks=200),
                               tol=1e-12, threads=4)
    G["sdd_running33_xi"] = xi
    G["sdd_running33_eta"] = eta
    # -- invert_mesh + quality_report (proj/src/invert.cpp, proj/src/quality.cpp)
    sx_, se_ = ref.solve_single_domain(B.density(B.RUNNING), UNIT, 33, 33, tol=1e-10)
    G["single_running33_xi"], G["single_running33_eta"] = sx_, se_
    X0, Y0 = ref.invert_mesh(sx_, se_, 33, 33, UNIT, 33, 33, threads=4)
    G["invert_single_running33"] = np.stack([X0, Y0])
    X1, Y1 = ref.invert_mesh(xi, eta, 33, 33, UNIT, 33, 33, threads=4)  # the SDD mesh above
    G["invert_sdd_running33"] = np.stack([X1, Y1])
    G["quality_sdd_running33"] = ref.quality(X1, Y1, 33, 33, UNIT, X0, Y0, B.density(B.RUNNING))
    X2, Y2 = ref.invert_mesh(sx_, se_, 33, 33, UNIT, 57, 41, threads=4)  # non-square target grid
    G["invert_single_running33_57x41"] = np.stack([X2, Y2])
    G["quality_single_running33_57x41"] = ref.quality(X2, Y2, 57, 41, UNIT)
    fx, fe = ref.solve_single_domain(B.density(B.FIVE_RING), FIVE, 41, 41, tol=1e-10)
    X3, Y3 = ref.invert_mesh(fx, fe, 41, 41, FIVE, 41, 41, threads=4)
    G["single_five41_xi"], G["single_five41_eta"] = fx, fe
    G["invert_single_five41"] = np.stack([X3, Y3])
    G["quality_single_five41"] = ref.quality(X3, Y3, 41, 41, FIVE)
    # -- perona_malik + smooth_interface (proj/src/smoothing.cpp)
    hx = 1.0 / 32
    dt_ok = 0.9 * hx * hx / 4.0
    for name, k, steps, scope in (("global", 1000.0, 5, 0), ("subdomain", 1000.0, 4, 1),
                                  ("edgestop", 0.5, 6, 0)):
        a, b = ref.perona_malik(xi, eta, 33, 33, UNIT, k, dt_ok, steps, scope, 2, 2)
        G[f"pm_{name}"] = np.stack([a, b])
    G["pm_dt"] = np.array([dt_ok])
    line = lines[0][0]  # a noisy interface line from solve_interfaces above
    G["loess_in"] = line
    for span in (3, 5, 9):
        G[f"loess_{span}"] = ref.smooth_interface(line, span)
    # 2x1: with crossing lines the reference's per-line smoothing breaks corner
    # agreement and solve_dirichlet raises ValidationError (mirrored in the tests)
    sxi, seta = ref.solve_sdd_smoothed(B.density(B.RUNNING), UNIT, 33, 33, 2, 1, 0, 0,
                                       B.walk_cfg(scheme="exp", lam=1000.0, seed=2, walks=300), 1e-12, 5)
    G["sdd_smoothed_running33"] = np.stack([sxi, seta])
    np.savez_compressed(OUT, **G)
    print(f"wrote {OUT}: {len(G)} arrays, {os.path.getsize(OUT) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()

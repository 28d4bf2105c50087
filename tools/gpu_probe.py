"""Development probe: parity + rough throughput on one B200 (run under gpurun)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1310_3435_b200 import sdd
from oracle import bindings as B

ctx = sdd.Context(0)
dom = sdd.RectDomain(0, 1, 0, 1)
odom = B.Domain(0, 1, 0, 1)
ref = B.Ref()
print("host threads", ref.hardware_threads(), flush=True)

def parity(kind, grad, cfg, ocfg, p, pid, n=2000, nx=65):
    m = sdd.MonitorFunction(kind, grad_mode=grad) if kind >= 16 else {0: sdd.MonitorFunction.constant(), 1: sdd.MonitorFunction.running_example()}[kind]
    spec = sdd.GridSpec(dom, nx, nx)
    bd = sdd.make_boundary_data(m, spec)
    t = time.time(); g = sdd.walk_dump(p, pid, m, dom, bd, cfg, 0, n, ctx=ctx); tg = time.time() - t
    tabs = ref.make_boundary(B.density(kind), odom, nx, nx)
    t = time.time(); r = ref.walk_dump(B.density(kind), odom, tabs, ocfg, p[0], p[1], pid, 0, n); tr = time.time() - t
    same = (g["steps"] == r["steps"]) & (g["edge"] == r["edge"]) & (g["epoch"] == r["epoch"])
    bit = (g["f"] == r["f"]) & (g["g"] == r["g"])
    df = np.max(np.abs(g["f"][same] - r["f"][same])) if same.any() else -1
    print(f"kind {kind} grad {grad} p {p}: struct-same {same.mean():.4f} bit-same {bit.mean():.4f} max|df| {df:.3e} "
          f"mean steps {g['steps'].mean():.1f}/{r['steps'].mean():.1f} gpu {tg:.3f}s ref {tr:.2f}s", flush=True)
    if not same.all():
        k = np.where(~same)[0][:3]
        print("  mismatches", g[k], r[k])

lin = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1, seed=1)
olin = B.walk_cfg(dt=1e-4, walks=1, seed=1)
parity(16, 0, lin, olin, (0.5, 0.5), 32 * 65 + 32)
parity(16, 0, lin, olin, (0.5, 2 / 64), 2 * 65 + 32)
parity(16, 1, lin, olin, (0.5, 0.5), 32 * 65 + 32)
parity(1, 0, lin, olin, (0.3, 0.6), 99)
ex = sdd.WalkConfig(scheme="exponential", lambda_=1000, walks=1, seed=3)
oex = B.walk_cfg(scheme="exp", lam=1000, walks=1, seed=3)
parity(1, 0, ex, oex, (0.3, 0.6), 99)
rs = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=1, seed=7, max_steps=300)
ors = B.walk_cfg(dt=1e-4, walks=1, seed=7, max_steps=300)
parity(0, 0, rs, ors, (0.02, 0.5), 1, n=400, nx=33)

# estimates vs reference, config-1 nodes, 2000 walks
m = sdd.MonitorFunction.ring()
spec = sdd.GridSpec(dom, 65, 65)
bd = sdd.make_boundary_data(m, spec)
pts = [(0.5, j / 64) for j in range(2, 63, 12)]
pids = [j * 65 + 32 for j in range(2, 63, 12)]
cfg = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=2000, seed=1)
e = sdd.mc_estimate_batch(pts, pids, m, dom, bd, cfg, ctx=ctx)
tabs = ref.make_boundary(B.density(16), odom, 65, 65)
t = time.time()
o = ref.mc_estimate_batch(B.density(16), odom, tabs, B.walk_cfg(dt=1e-4, walks=2000, seed=1),
                          [p[0] for p in pts], [p[1] for p in pts], pids, threads=0)
print("ref est time", time.time() - t)
print("xi gpu", e["xi"], "\nxi ref", o["xi"], "\ndiff", e["xi"] - o["xi"], "\nse", o["se_xi"])
print("bit-equal xi:", (e["xi"] == o["xi"]).mean(), "edge hits equal:", (e["edge_hits"] == o["edge_hits"]).all())

# throughput: config 1 full (61 nodes x 1e4), fp64 FD and analytic, then config-2-like
def tput(mm, cfgx, nodes, pids_, label):
    sdd.mc_estimate_batch(nodes[:4], pids_[:4], mm, dom, bd, cfgx, ctx=ctx)
    t = time.time()
    r = sdd.mc_estimate_batch(nodes, pids_, mm, dom, bd, cfgx, ctx=ctx)
    wall = time.time() - t
    st = ctx.last_stats()
    print(f"{label}: {len(nodes)} nodes x {cfgx.walks} walks: steps {st['path_steps']:.4e} kernel {st['kernel_ms']:.1f} ms "
          f"wall {wall:.3f}s -> {st['path_steps'] / (st['kernel_ms'] / 1e3):.4e} path-steps/s", flush=True)
    return r

lay = sdd.build_layout(spec, 2, 2)
plan = sdd.plan_interface_points("equispaced", 31, m, lay)
nodes, pids_ = [], []
for line, ps in zip(lay.lines, plan.stochastic):
    for p in ps:
        i, j = (line.fixed_index, p) if line.vertical else (p, line.fixed_index)
        if j * 65 + i not in pids_:
            nodes.append(spec.node(i, j)); pids_.append(j * 65 + i)
print("config-1 mc nodes", len(nodes))
c1 = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=10000, seed=1)
tput(m, c1, nodes, pids_, "cfg1 fp64 FD(ref)")
tput(sdd.MonitorFunction.ring(analytic=True), c1, nodes, pids_, "cfg1 fp64 analytic")
c1f = sdd.WalkConfig(scheme="linear", dt=1e-4, walks=10000, seed=1, precision="fp32")
tput(sdd.MonitorFunction.ring(analytic=True), c1f, nodes, pids_, "cfg1 fp32 analytic")
# config 2 sized: 129^2 4x4 all -> 753 nodes, 1e4 walks slab, dt=2e-5
spec2 = sdd.GridSpec(dom, 129, 129)
bd2 = sdd.make_boundary_data(m, spec2)
lay2 = sdd.build_layout(spec2, 4, 4)
nodes2, pids2 = [], []
for line in lay2.lines:
    for p in range(1, 128):
        i, j = (line.fixed_index, p) if line.vertical else (p, line.fixed_index)
        if j * 129 + i not in pids2:
            nodes2.append(spec2.node(i, j)); pids2.append(j * 129 + i)
print("config-2 nodes", len(nodes2))
bd = bd2
c2 = sdd.WalkConfig(scheme="linear", dt=2e-5, walks=2000, seed=1)
tput(sdd.MonitorFunction.ring(analytic=True), c2, nodes2, pids2, "cfg2 slab fp64 analytic")
tput(m, c2, nodes2, pids2, "cfg2 slab fp64 FD(ref)")
c2f = sdd.WalkConfig(scheme="linear", dt=2e-5, walks=2000, seed=1, precision="fp32")
tput(sdd.MonitorFunction.ring(analytic=True), c2f, nodes2, pids2, "cfg2 slab fp32 analytic")

# solver parity
w = ref.weight_values(B.density(16), odom, 33, 33)
tb = ref.make_boundary(B.density(16), odom, 33, 33)
for method in ("jacobi", "rbsor"):
    for tol in (1e-10, 1e-13):
        ur, itr, fur, cvr = ref.solve_dirichlet(w, 33, 33, 1 / 32, 1 / 32, *tb.f, tol=tol)
        bc = sdd.EdgeData(*tb.f)
        t = time.time()
        s = sdd.solve_dirichlet(w, 33, 33, 1 / 32, 1 / 32, bc, sdd.SolverConfig(tol=tol, method=method), ctx=ctx)
        print(f"solver {method} tol {tol}: iters gpu {s.iterations} ref {itr} max|du| {np.max(np.abs(s.values - ur)):.3e} "
              f"bit-equal {(s.values == ur).all()} time {time.time() - t:.3f}s kernel {ctx.last_stats()['kernel_ms']:.2f} ms")

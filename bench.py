"""Benchmark: SDE walk path-steps/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
unit square, 129x129 global grid split 4x4, every interior node of the six
interface lines (753 unique Monte Carlo nodes), ring density w with the
analytic drift grad(w)/w, Euler-Maruyama dt = 2e-5 with the reference's
Brownian-bridge exit test, fp64.  One bench step = the whole walk phase of
config 2's solve_interfaces: all 753 nodes at the config's 10^5 paths per node
(~6.2e11 path-steps; the seed changes every step).

  value  : path-steps/s, device-resident inputs (sddg_mc_estimate_batch_device),
           CUDA events on the launching stream, max over ranks, L2 flushed
           (256 MiB write) before every timed step.
  e2e    : the same metric through the public host-buffer API
           (sdd.mc_estimate_batch -> sddg_mc_estimate_batch), pinned host
           inputs copied in and estimates copied out every step, wall clock.
  roofline: walk kernel (K1): instruction issue (thread-
           instructions of this launch / K1 event time over SMs x 128 per clock)
           with the FP64 pipe beside it; "census" is the cross-check (algorithmic
           DP flops per path-step x path-steps / K1 event time against the DFMA
           peak measured on this GPU by sddg_probe_fma_peak).
  cpu_baseline: the reference's own mc_estimate (oracle/_ref, built from
           /root/reference/proj/src) on all host threads over a fixed node
           subsample of the same workload.

--workload config3 runs BASELINE's multi-GPU scaling run instead (1025^2, 8x8,
shock density, 14,273 nodes, fp32 walks with fp64 sums; --walks paths per node
per step, default 10,000 of the config's 1e6), with the same timing, roofline
(issue slots; fp32) and, under torchrun, the same sharded path.

--impl reference runs the reference CPU implementation alone (rank 0), each
step a bounded sample of the workload, and prints the same metric.
Multi-GPU (torchrun, one process per GPU): strong scaling of the same
workload through the library's multi-GPU context (sddg_create_dist): the 753
nodes are sharded across the ranks by expected cost (sddg_shard_plan) and
every step ends with the one ncclAllGather of the 128-B estimate records
inside the timed region, so every rank holds all 753 estimates.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GRID, SUBS, DT, WALKS_PER_STEP, CONFIG_WALKS = 129, 4, 2e-5, 100_000, 100_000
# naive census of FP64 operations per interior path-step (transcendental = 1),
# SURVEY.md 8(d) / DESIGN.md "Roofline"
DP_FLOPS_PER_STEP = 57
CPU_SAMPLE_STRIDE, CPU_SAMPLE_WALKS = 24, 2000  # every 24th node (32 nodes) x 2000 walks


def config2_nodes():
    """Unique interface nodes of the 129^2 4x4 layout in solve_interfaces order
    (vertical lines first, proj/src/decomposition.cpp:44-51,156-169)."""
    h = 1.0 / (GRID - 1)
    seen, px, py, pid = set(), [], [], []
    block = (GRID - 1) // SUBS
    lines = [(True, a * block) for a in range(1, SUBS)] + [(False, b * block) for b in range(1, SUBS)]
    for vertical, fixed in lines:
        for p in range(1, GRID - 1):
            i, j = (fixed, p) if vertical else (p, fixed)
            g = j * GRID + i
            if g in seen:
                continue
            seen.add(g)
            px.append(0.0 + i * h)
            py.append(0.0 + j * h)
            pid.append(g)
    return np.array(px), np.array(py), np.array(pid, np.uint64)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[4 + k].lower() == "active"})
        power = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(power) if power else None}


def pipe_fractions(steps_per_s, sm_mhz, precision, sms):
    """Issue-slot and FP64-pipe fractions of K1, live: the static SASS count of
    one step (profiles/sass_walk_step.json, tools/sass_trace.py) x the measured
    path-steps/s, over the SM's issue rate (4 warp-instructions/clk = 128
    thread-instructions) and FP64 rate (64 lanes/clk) at the sampled clock.
    These count useful (active-lane) work only."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "sass_walk_step.json")))
        k = d["fp64_ring" if precision == "fp64" else "fp32_shock"]
        hz = (sm_mhz or 0) * 1e6
        if not hz:
            return None
        out = {"sass_instructions_per_step": k["instructions_per_step"],
               "issue_frac": k["instructions_per_step"] * steps_per_s / (sms * 128 * hz),
               "source": "profiles/sass_walk_step.json (cuobjdump trace of the hot step) x live "
                         "path-steps/s / (SMs x 128 thread-instr/clk x sampled SM clock)"}
        if precision == "fp64":
            out["sass_fp64_per_step"] = k["fp64_per_step"]
            out["fp64_pipe_frac"] = k["fp64_per_step"] * steps_per_s / (sms * 64 * hz)
        return out
    except (OSError, KeyError, ValueError, TypeError):
        return None


def ncu_summary():
    """Pipe / issue utilisation of K1 from the committed ncu capture at the
    bench config (profiles/ncu_walk_summary.json; measured with ncu, not in
    this run)."""
    path = os.path.join(ROOT, "profiles", "ncu_walk_summary.json")
    try:
        d = json.load(open(path))["fp64_config2_1e5"]
        m = d["metrics"]
        g = lambda k: float(m[k]["value"])  # noqa: E731
        return {"source": "profiles/ncu_walk_summary.json fp64_config2_1e5 (" + d["command"] + ")",
                "issue_slots_busy_pct": g("sm__inst_issued.avg.pct_of_peak_sustained_active"),
                "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "alu_pipe_pct": g("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                "active_lanes_per_warp_instruction": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
                "instructions_per_path_step": d["instructions_per_path_step"],
                "dram_bytes_per_walk": d.get("dram_bytes_per_walk")}
    except (OSError, KeyError, ValueError):
        return None


def traffic_per_launch(walks):
    s = ncu_summary()
    if not s or not s.get("dram_bytes_per_walk"):
        return None
    return s["dram_bytes_per_walk"] * walks


def cpu_reference_sample(ref, B, threads, walks=CPU_SAMPLE_WALKS, seed=1):
    """The reference's mc_estimate (FD ring drift -- its only route for a
    user density) over the fixed node subsample; returns (path-steps, seconds)."""
    px, py, pid = config2_nodes()
    sel = slice(0, None, CPU_SAMPLE_STRIDE)
    dom = B.Domain(0, 1, 0, 1)
    d = B.density(B.RING_W)
    tabs = ref.make_boundary(d, dom, GRID, GRID)
    cfg = B.walk_cfg(dt=DT, walks=walks, seed=seed)
    t0 = time.perf_counter()
    ref.mc_estimate_batch(d, dom, tabs, cfg, px[sel], py[sel], pid[sel], threads=threads)
    sec = time.perf_counter() - t0
    # path-steps of the identical walks (same streams): counted by the C
    # restatement, which is bit-identical to the reference (tests/test_oracle_pins.py)
    return sec, (px[sel], py[sel], pid[sel], tabs, cfg)


def count_steps(B, sample, threads):
    px, py, pid, tabs, cfg = sample
    orc = B.Oracle()
    e = orc.mc_estimate_batch(B.density(B.RING_W), B.Domain(0, 1, 0, 1), tabs, cfg, px, py, pid,
                              threads=threads)
    return int(e["path_steps"].sum())


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import bindings as B
    try:
        B.ensure_built()
        ref = B.Ref()
    except Exception as exc:  # the reference library could not be loaded
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref: {exc}"}))
        return 0
    threads = ref.hardware_threads()
    walks = CPU_SAMPLE_WALKS // 2
    times, sample = [], None
    for k in range(args.warmup + args.steps):
        # the same bounded sample every step (identical work per step)
        sec, sample = cpu_reference_sample(ref, B, threads, walks=walks, seed=1)
        if k >= args.warmup:
            times.append(sec)
    # path-steps of those walks, counted once by the bit-identical C restatement
    steps = [count_steps(B, sample, threads)] * len(times)
    value = float(sum(steps) / sum(times))
    n_nodes = len(range(0, 753, CPU_SAMPLE_STRIDE))
    sample_desc = (f"config-2 walk phase sample: every {CPU_SAMPLE_STRIDE}th of the 753 interface "
                   f"nodes ({n_nodes} nodes) x {walks} paths, dt={DT}, ring density via the "
                   f"reference's user_supplied FD drift")
    print(json.dumps({
        "impl": "reference", "metric": "SDE walk path-steps/s", "value": value,
        "unit": "path-steps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "BASELINE config 2 walk phase (129^2, 4x4, ring, dt=2e-5), bounded sample",
                   "nodes": n_nodes, "paths_per_node": walks},
        "cpu_baseline": {"value": value, "unit": "path-steps/s", "cores": threads,
                         "kind": "reference", "sample": sample_desc},
        "e2e": {"value": value, "unit": "path-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))
    return 0


def hbm_peak_gbs():
    """Measured HBM copy bandwidth (driver-written MEASURED_PEAKS.json), else
    the profiling recipe's B200 figure."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 7700.0, "fallback: B200 nominal 7.7 TB/s"


def solver_rooflines(sdd, ctx):
    g, subs_n = 1025, 8
    spec = sdd.GridSpec(sdd.RectDomain(0.0, 1.0, 0.0, 1.0), g, g)
    lay = sdd.build_layout(spec, subs_n, subs_n)
    bxy = lay.block_x + 1
    x = np.linspace(0.0, 1.0, g)
    X, Y = np.meshgrid(x, x)
    w = (1.0 + 20.0 / np.cosh(50 * (Y - 0.5 - 0.15 * np.sin(2 * np.pi * X))) ** 2).ravel()
    peak, src = hbm_peak_gbs()
    onchip = ctx.probe_onchip_bandwidth()
    out = {"bytes_per_point_update": 40, "peak_GBps": peak, "peak_source": src,
           "onchip_peaks_GBps": onchip,
           "onchip_note": "the batches stay on chip (SURVEY D9): K3 reads its 32 B of packed weights per "
                          "update from L2 (u in shared memory) -> frac_of_l2; K3c keeps weights and u in "
                          "shared memory: 80 B of shared-memory reads per update (5 u + 32 B weights + "
                          "the write) -> frac_of_smem; peaks measured on this GPU (sddg_probe_onchip_bandwidth)"}
    for name, n_jobs in (("config3_batch", 128), ("batch_2048", 2048)):
        rng = np.random.default_rng(3)
        jobs, bcs = [], []
        for s_ in range(n_jobs):
            q = s_ % lay.subdomain_count()
            jobs.append(lay.subdomain(q % subs_n, q // subs_n))
            v = np.sort(rng.random(4))
            e = lambda a, b: np.linspace(a, b, bxy)  # noqa: E731
            bcs.append(sdd.EdgeData(e(v[0], v[1]), e(v[2], v[3]), e(v[0], v[2]), e(v[1], v[3])))
        cfg = sdd.SolverConfig(tol=1e-10, method="rbsor")
        best = None
        for _ in range(3):
            res = sdd.solve_dirichlet_batch(w, g, g, 1 / (g - 1), 1 / (g - 1), jobs, bcs, cfg, ctx=ctx)
            ms = ctx.last_stats()["kernel_ms"]
            best = ms if best is None else min(best, ms)
        its = np.array([r.iterations for r in res])
        upd = float(its.sum()) * (bxy - 2) ** 2
        gbs = upd * 40 / (best / 1e3) / 1e9
        out[name] = {"solves": n_jobs, "grid": f"{bxy}^2", "kernel": "K3c (cluster per solve)" if n_jobs <= 148
                     else "K3 (CTA per solve)", "ms": best, "sweeps_mean": float(its.mean()),
                     "sweeps_max": int(its.max()), "point_updates_per_s": upd / (best / 1e3),
                     "effective_GBps": gbs, "frac_of_hbm_peak": gbs / peak,
                     "converged": bool(all(r.converged for r in res))}
        ups = upd / (best / 1e3)
        if n_jobs <= 148:
            out[name]["onchip_bound"] = "smem"
            out[name]["frac_of_smem"] = ups * 80 / 1e9 / onchip["smem_GBps"]
        else:
            out[name]["onchip_bound"] = "l2"
            out[name]["frac_of_l2"] = ups * 32 / 1e9 / onchip["l2_GBps"]
    return out


# ---------------------------------------------------------------- paper table
# `python bench.py --paper-table`: the reference's own end-to-end workload --
# the paper's timing table as the
# reference's acceptance criterion c11 runs it (proj/tests/acceptance.cpp:
# 331-372): five-ring density on [-1,1]^2, 4x4 subdomains, optimal interface
# placement, exponential stepping (lambda 1000), N = 5000 walks per node,
# seed 1, tol 1e-8, grids 37^2 ... 197^2.  Per grid: T_stoc / T_sub / T_total
# of solve_sdd and T_1 of the single-domain solve -- ours (reference-mode
# drift with the reference Jacobi or RB-SOR, and the performance-mode
# five-ring drift with RB-SOR) and, as this mode's CPU-baseline leg, the
# reference's (oracle/_ref on every host thread; T_1 sequential as in c11) --
# plus the largest difference between the meshes.  One JSON object
# (profiles/r01_paper_table.json).
PAPER_GRIDS = (37, 77, 117, 157, 197)


def _paper_ours(sdd, m, n, ctx, solver):
    spec = sdd.GridSpec(m.domain, n, n)
    lay = sdd.build_layout(spec, 4, 4)
    plan = sdd.plan_interface_points("optimal", 0, m, lay)
    cfg = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=5000, seed=1)
    scfg = sdd.SolverConfig(tol=1e-8, method=solver)
    sdd.solve_sdd(m, lay, plan, cfg, scfg, ctx=ctx)  # warm-up (module load, buffers)
    t0 = time.perf_counter()
    r = sdd.solve_sdd(m, lay, plan, cfg, scfg, ctx=ctx)
    wall = time.perf_counter() - t0
    lay1 = sdd.build_layout(spec, 1, 1)
    plan1 = sdd.plan_interface_points("all", 0, m, lay1)
    t0 = time.perf_counter()
    single = sdd.solve_sdd(m, lay1, plan1, sdd.WalkConfig(walks=1), scfg, ctx=ctx)
    t_1 = time.perf_counter() - t0
    mesh = sdd.invert_mesh(r.xi, r.eta, spec, n, n, ctx=ctx)
    ref = sdd.invert_mesh(single.xi, single.eta, spec, n, n, ctx=ctx)
    q = sdd.quality_report(mesh, ref, m, ctx=ctx)
    return r, {"t_stoc_s": r.t_stoc, "t_sub_s": r.t_sub, "t_total_s": r.t_stoc + r.t_sub + r.t_smooth,
               "wall_s": wall, "t_1_s": t_1, "mc_points": r.mc_points, "path_steps": r.path_steps,
               "path_steps_per_s": r.path_steps / r.t_stoc if r.t_stoc > 0 else None,
               "r_mean": q.r_mean, "q_max": q.q_max, "solver": solver}


def _paper_reference(n, threads, with_t1):
    from oracle import bindings as B  # the CPU-baseline leg of this mode
    ref = B.Ref()
    dens, dom = B.density(B.FIVE_RING), B.Domain(-1.0, 1.0, -1.0, 1.0)
    cfg = B.walk_cfg(scheme="exponential", lam=1000.0, walks=5000, seed=1)
    xi, eta, t = ref.solve_sdd(dens, dom, n, n, 4, 4, 2, 0, cfg, tol=1e-8, threads=threads)
    out = {"t_stoc_s": t[0], "t_sub_s": t[1], "t_total_s": float(t.sum()), "threads": threads}
    if with_t1:
        t0 = time.perf_counter()
        ref.solve_single_domain(dens, dom, n, n, tol=1e-8)
        out["t_1_s"] = time.perf_counter() - t0
    return xi, eta, out


# ------------------------------------------------------------ CPU configs
# `python bench.py --cpu-configs`: the reference CPU build's walk rate on every
# BASELINE config: config 1 in full, configs 2-5 on a fixed
# deterministic node subsample with the config's dt and density (the
# reference's user_supplied FD drift, its only route for these densities), all
# host threads.  Reports path-steps/s, mean steps per path and the CPU seconds
# the full config would take at that rate.  One JSON object
# (profiles/r01_cpu_configs.json); the GPU side of each row is measured by
# tools/config_sweep.py / tools/config3_full.py and this bench.
CPU_CONFIGS = (
    # name, density, grid, layout, placement, k, dt, paths per node, node stride, sample paths
    ("config1", "ring", 65, 2, "equispaced", 31, 1e-4, 10_000, 1, 10_000),
    ("config2", "ring", 129, 4, "all", 0, 2e-5, 100_000, 24, 2_000),
    ("config3", "shock", 1025, 8, "all", 0, 1e-5, 1_000_000, 476, 2_000),
    ("config4", "two-bump", 513, 4, "equidistributed", 32, 1e-5, 200_000, 8, 1_000),
    ("config5", "ring", 0, 0, "", 0, 1e-5, 1_000_000, 128, 1_000),
)


def cpu_configs(args):
    from oracle import bindings as B  # this mode is a CPU-baseline leg
    from paper_1310_3435_b200 import sdd
    B.ensure_built()
    ref, orc = B.Ref(), B.Oracle()
    threads = ref.hardware_threads()
    kinds = {"ring": (B.RING_W, sdd.RING_W), "shock": (B.SHOCK_W, sdd.SHOCK_W),
             "two-bump": (B.TWOBUMP_W, sdd.TWOBUMP_W)}
    out = {"threads": threads, "drift": "reference user_supplied FD of rho = 1/w (h = 1e-6)",
           "configs": {}}
    for name, dens, grid, subs, place, k, dt, paths, stride, sample_paths in CPU_CONFIGS:
        bk, sk = kinds[dens]
        m = sdd.MonitorFunction.weight(sk)
        dom = B.Domain(0, 1, 0, 1)
        if name == "config5":
            pts = np.clip(np.random.default_rng(1).uniform(0.0, 1.0, (4096, 2)), 1e-9, 1 - 1e-9)
            px, py, pid = pts[:, 0].copy(), pts[:, 1].copy(), np.arange(4096, dtype=np.uint64)
            grid = 129
        else:
            lay = sdd.build_layout(sdd.GridSpec(sdd.RectDomain(0, 1, 0, 1), grid, grid), subs, subs)
            px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points(place, k, m, lay))
        n_nodes = len(px)
        sel = slice(0, None, stride)
        d = B.density(bk)
        tabs = ref.make_boundary(d, dom, grid, grid)
        cfg = B.walk_cfg(dt=dt, walks=sample_paths, seed=1)
        t0 = time.perf_counter()
        ref.mc_estimate_batch(d, dom, tabs, cfg, px[sel], py[sel], pid[sel], threads=threads)
        sec = time.perf_counter() - t0
        # path-steps of the same walks, counted by the bit-identical C restatement
        steps = int(orc.mc_estimate_batch(d, dom, tabs, cfg, px[sel], py[sel], pid[sel],
                                          threads=threads)["path_steps"].sum())
        n_sel = len(px[sel])
        per_path = steps / (n_sel * sample_paths)
        rate = steps / sec
        out["configs"][name] = {
            "nodes": n_nodes, "paths_per_node": paths, "dt": dt, "density": dens,
            "sample": f"every {stride}th node ({n_sel}) x {sample_paths} paths",
            "sample_path_steps": steps, "sample_seconds": sec, "path_steps_per_s": rate,
            "mean_steps_per_path": per_path,
            "full_config_path_steps_est": per_path * n_nodes * paths,
            "full_config_cpu_seconds_est": per_path * n_nodes * paths / rate}
        print(name, json.dumps(out["configs"][name]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))
    return 0


def paper_table(args):
    from paper_1310_3435_b200 import sdd
    ctx = sdd.Context(0)
    m = sdd.MonitorFunction.five_ring()
    m_fast = sdd.MonitorFunction.five_ring(analytic=True)  # performance-mode drift
    threads = os.cpu_count() or 1
    rows = {}
    for n in PAPER_GRIDS:
        r, row = _paper_ours(sdd, m, n, ctx, "jacobi")
        _, row_sor = _paper_ours(sdd, m, n, ctx, "rbsor")
        rf, row_fast = _paper_ours(sdd, m_fast, n, ctx, "rbsor")
        rows[n] = {"ours": row, "ours_rbsor": row_sor, "ours_fast_rbsor": row_fast}
        if not args.no_cpu_baseline:
            xi, eta, rr = _paper_reference(n, threads, n <= 157)
            rows[n]["reference_cpu"] = rr
            rows[n]["max_abs_mesh_diff"] = float(max(np.max(np.abs(xi - r.xi)), np.max(np.abs(eta - r.eta))))
            rows[n]["max_abs_mesh_diff_fast"] = float(max(np.max(np.abs(xi - rf.xi)),
                                                          np.max(np.abs(eta - rf.eta))))
            rows[n]["t_total_speedup"] = rr["t_total_s"] / row["t_total_s"]
            rows[n]["t_total_speedup_fast"] = rr["t_total_s"] / row_fast["t_total_s"]
        print(n, json.dumps(rows[n]), file=sys.stderr, flush=True)
    readme = readme_workloads(sdd, ctx, threads, not args.no_cpu_baseline)
    print(json.dumps({"workload": "paper table / acceptance c11: five-ring on [-1,1]^2, 4x4, optimal placement, "
                      "exponential lambda 1000, N 5000, seed 1, tol 1e-8", "host_threads": threads,
                      "grids": rows, "readme_workloads": readme}, indent=1))
    return 0


def readme_workloads(sdd, ctx, threads, with_ref):
    """The reference README's CLI examples (proj/README.md:68-79) on the
    running-example density, 29^2 grid, seed 1: `stochastic-full` (every
    interior node, N = 10000, exponential:1000) and `sdd` (2x2, optimal
    placement, N = 10000, exponential:10000); ours on the GPU (reference-mode
    drift, the reference Jacobi) vs the reference CPU build."""
    m = sdd.MonitorFunction.running_example()
    spec = sdd.GridSpec(sdd.RectDomain(0, 1, 0, 1), 29, 29)
    out = {}
    cfg = sdd.WalkConfig(scheme="exponential", lambda_=1000.0, walks=10_000, seed=1)
    sdd.stochastic_full(m, spec, cfg, ctx=ctx)
    t0 = time.perf_counter()
    xi, eta, st = sdd.stochastic_full(m, spec, cfg, ctx=ctx)
    row = {"gpu_s": time.perf_counter() - t0, "mc_points": st["mc_points"]}
    if with_ref:
        from oracle import bindings as B  # CPU-baseline leg
        ref = B.Ref()
        dom = B.Domain(0, 1, 0, 1)
        d = B.density(B.RUNNING)
        tabs = ref.make_boundary(d, dom, 29, 29)
        ids = [(i, j) for j in range(1, 28) for i in range(1, 28)]
        t0 = time.perf_counter()
        e = ref.mc_estimate_batch(d, dom, tabs, B.walk_cfg(scheme="exponential", lam=1000.0, walks=10_000, seed=1),
                                  [0.0 + i * (1.0 / 28) for i, _ in ids], [0.0 + j * (1.0 / 28) for _, j in ids],
                                  [j * 29 + i for i, j in ids],  # GridSpec::node = min + i h
                                  threads=threads)
        row["reference_cpu_s"] = time.perf_counter() - t0
        row["speedup"] = row["reference_cpu_s"] / row["gpu_s"]
        pid = np.array([j * 29 + i for i, j in ids])
        row["max_abs_diff_xi"] = float(np.max(np.abs(xi[pid] - e["xi"])))
    out["stochastic_full_running_29"] = row
    lay = sdd.build_layout(spec, 2, 2)
    plan = sdd.plan_interface_points("optimal", 0, m, lay)
    wc = sdd.WalkConfig(scheme="exponential", lambda_=10_000.0, walks=10_000, seed=1)
    sc = sdd.SolverConfig(tol=1e-8)
    sdd.solve_sdd(m, lay, plan, wc, sc, ctx=ctx)
    t0 = time.perf_counter()
    r = sdd.solve_sdd(m, lay, plan, wc, sc, ctx=ctx)
    row = {"gpu_s": time.perf_counter() - t0, "t_stoc_s": r.t_stoc, "t_sub_s": r.t_sub, "mc_points": r.mc_points}
    if with_ref:
        t0 = time.perf_counter()
        rxi, reta, rt = ref.solve_sdd(d, dom, 29, 29, 2, 2, 2, 0,
                                      B.walk_cfg(scheme="exponential", lam=10_000.0, walks=10_000, seed=1),
                                      tol=1e-8, threads=threads)
        row["reference_cpu_s"] = time.perf_counter() - t0
        row["speedup"] = row["reference_cpu_s"] / row["gpu_s"]
        row["max_abs_mesh_diff"] = float(max(np.max(np.abs(rxi - r.xi)), np.max(np.abs(reta - r.eta))))
    out["sdd_running_29_2x2"] = row
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2", choices=["config2", "config3"],
                    help="config2: the metric's config (default); config3: BASELINE's multi-GPU scaling run "
                         "(1025^2, 8x8, shock, 14,273 nodes, fp32 walks), --walks paths per node per step")
    ap.add_argument("--precision", default=None, choices=["fp64", "fp32"])
    ap.add_argument("--drift", default="analytic", choices=["analytic", "reference"])
    ap.add_argument("--walks", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-mesh", action="store_true", help="skip the end-to-end mesh-gen timings")
    ap.add_argument("--no-solver", action="store_true", help="skip the subdomain-solver roofline")
    ap.add_argument("--cpu-configs", action="store_true",
                    help="the reference CPU walk rate on every BASELINE config (CPU only)")
    ap.add_argument("--paper-table", action="store_true",
                    help="the reference's own workload (paper table / acceptance c11) vs the reference CPU")
    args = ap.parse_args()
    c3 = args.workload == "config3"
    if args.precision is None:
        args.precision = "fp32" if c3 else "fp64"
    if args.walks is None:
        args.walks = 10_000 if c3 else WALKS_PER_STEP
    if c3:  # the config-2 side measurements do not apply
        args.no_mesh = args.no_solver = args.no_cpu_baseline = True
    if args.impl == "reference":
        return run_reference(args)
    if args.paper_table:
        return paper_table(args)
    if args.cpu_configs:
        return cpu_configs(args)

    import torch
    import torch.distributed as dist
    from paper_1310_3435_b200 import sdd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    cdev = "cuda"  # device of the timing collectives
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # the library's own communicator over the same ranks (sddg_create_dist)
        nid = [sdd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        ctx = sdd.Context.dist(local, rank, world, nid[0])
        print(f"sddg team: {json.dumps(ctx.team_info())} on cuda:{local}", file=sys.stderr, flush=True)
    elif os.environ.get("SDDG_BENCH_TEAM"):  # the multi-GPU code path over a one-rank communicator
        ctx = sdd.Context.dist(local, 0, 1, sdd.nccl_unique_id())
        print(f"sddg team: {json.dumps(ctx.team_info())} on cuda:{local}", file=sys.stderr, flush=True)
    else:
        ctx = sdd.Context(local)
    stream = torch.cuda.current_stream()

    dom = sdd.RectDomain(0.0, 1.0, 0.0, 1.0)
    if c3:
        # BASELINE config 3: 1025^2 grid split 8x8, shock-layer density, every
        # interior node of the 14 interface lines, dt = 1e-5, fp32 walks
        m = sdd.MonitorFunction.shock(analytic=args.drift == "analytic")
        grid, dt_w, config_walks = 1025, 1e-5, 1_000_000
        spec = sdd.GridSpec(dom, grid, grid)
        lay3 = sdd.build_layout(spec, 8, 8)
        px, py, pid = sdd.interface_nodes(m, lay3, sdd.plan_interface_points("all", 0, m, lay3))
        pid = np.asarray(pid, dtype=np.uint64)
        workload = ("BASELINE config 3 walk phase: 1025^2 grid, 8x8 subdomains, all 14,273 interface nodes, "
                    "shock-layer density (analytic grad w / w), linear EM dt=1e-5 + bridge exit test; one step "
                    f"= {args.walks} of the config's 1e6 paths per node")
    else:
        m = sdd.MonitorFunction.ring(analytic=args.drift == "analytic")
        grid, dt_w, config_walks = GRID, DT, CONFIG_WALKS
        spec = sdd.GridSpec(dom, GRID, GRID)
        px, py, pid = config2_nodes()
        workload = ("BASELINE config 2 walk phase (one step = the full config): 129^2 "
                    "grid, 4x4 subdomains, all 753 interface nodes x 1e5 paths, ring "
                    "density (analytic grad w / w), linear EM dt=2e-5 + bridge exit test")
    bd = sdd.make_boundary_data(m, spec)
    n = len(px)
    d_px = torch.tensor(px, dtype=torch.float64, device="cuda")
    d_py = torch.tensor(py, dtype=torch.float64, device="cuda")
    d_pid = torch.tensor(pid.astype(np.int64), dtype=torch.int64, device="cuda")
    d_out = torch.empty(n * sdd.ESTIMATE_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def cfg_for(step):
        return sdd.WalkConfig(scheme="linear", dt=dt_w, walks=args.walks, seed=1 + step,
                              precision=args.precision)

    def one_step(step):
        sdd.mc_estimate_batch_device(d_px, d_py, d_pid, d_out, m, dom, bd, cfg_for(step), ctx=ctx,
                                     stream=stream)
        return ctx.last_stats()

    for k in range(args.warmup):
        one_step(k)
    torch.cuda.synchronize()

    peak_fp64 = ctx.probe_fma_peak("fp64")
    peak_fp32 = ctx.probe_fma_peak("fp32")

    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    total_steps, k1_ms, launches = 0, 0.0, 0
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record(stream)
        st = one_step(args.warmup + k)
        ev[k][1].record(stream)
        total_steps += st["path_steps"]
        k1_ms += st["kernel_ms"]
        launches += st["launches"]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = sum(a.elapsed_time(b) for a, b in ev)
    # path-steps: every rank holds all records after the all-gather, so
    # total_steps already counts the whole job; time: max over ranks
    all_steps = float(total_steps)
    shard_k1 = None
    if world > 1:
        t = torch.tensor([elapsed_ms, k1_ms], dtype=torch.float64, device=cdev)
        tall = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(tall, t)
        elapsed_ms = max(float(v[0]) for v in tall)
        shard_k1 = [float(v[1]) / args.steps for v in tall]
    value = all_steps / (elapsed_ms / 1e3)

    # ---- e2e through the public host-buffer API (pinned inputs, D2H result)
    e2e = None
    if not args.no_e2e:
        pts = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
        pts[:, 0] = torch.from_numpy(px)
        pts[:, 1] = torch.from_numpy(py)
        hpid = torch.from_numpy(pid.astype(np.int64)).pin_memory()
        sdd.mc_estimate_batch(pts.numpy(), hpid.numpy().view(np.uint64), m, dom, bd, cfg_for(0), ctx=ctx)
        e_steps, e_sec = 0, 0.0
        for k in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sdd.mc_estimate_batch(pts.numpy(), hpid.numpy().view(np.uint64), m, dom, bd,
                                  cfg_for(args.warmup + k), ctx=ctx)
            e_sec += time.perf_counter() - t0
            e_steps += ctx.last_stats()["path_steps"]
        if world > 1:
            et = torch.tensor([e_sec], dtype=torch.float64, device=cdev)
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
            e_sec = float(et[0])
        tables_bytes = 8 * 4 * (grid + grid)
        e2e = {"value": e_steps / e_sec, "unit": "path-steps/s",
               "h2d_bytes_per_step": int(n * 24 + tables_bytes),
               "d2h_bytes_per_step": int(n * sdd.ESTIMATE_DTYPE.itemsize),
               "api": "sdd.mc_estimate_batch -> sddg_mc_estimate_batch (host buffers)"}

    # ---- end-to-end mesh generation (T_stoc + T_sub, proj/src/cli.cpp:322):
    # full BASELINE configs 1 and 2 through sdd.solve_sdd, once each (every
    # rank calls it: with several GPUs the nodes and subdomains are sharded)
    mesh = None
    if not args.no_mesh:
        mesh = {}
        for name, grid, subs_, place, k, walks, dt in (("config1", 65, 2, "equispaced", 31, 10_000, 1e-4),
                                                       ("config2", 129, 4, "all", 0, 100_000, 2e-5)):
            lay = sdd.build_layout(sdd.GridSpec(dom, grid, grid), subs_, subs_)
            plan = sdd.plan_interface_points(place, k, m, lay)
            wc = sdd.WalkConfig(scheme="linear", dt=dt, walks=walks, seed=1, precision=args.precision)
            sc = sdd.SolverConfig(tol=1e-10, method="rbsor")
            # warm-up with 1,000 paths per node (module loads, buffers of this shape)
            sdd.solve_sdd(m, lay, plan, sdd.WalkConfig(scheme="linear", dt=dt, walks=1000, seed=2,
                                                       precision=args.precision), sc, ctx=ctx)
            r = sdd.solve_sdd(m, lay, plan, wc, sc, ctx=ctx)
            mesh[name] = {"t_stoc_s": r.t_stoc, "t_sub_s": r.t_sub, "t_total_s": r.t_stoc + r.t_sub,
                          "mc_points": r.mc_points, "paths_per_node": walks,
                          "path_steps": r.path_steps, "subdomain_solves": r.subdomain_solves,
                          "solver": "rbsor tol 1e-10", "gpus": world}

    # ---- like-for-like with the reference arm: the full config-2 walk phase
    # (753 nodes x 1e5 paths) with the reference's own drift (user_supplied
    # central difference of rho = 1/w, monitor.cpp:206-219; the bit-faithful
    # parity mode, what a drop-in caller gets by default), end to end through
    # the public host-buffer API, one launch after a short warm-up launch
    parity_mode = None
    if rank == 0 and world == 1 and not args.no_mesh and args.drift == "analytic" and not c3:
        m_ref = sdd.MonitorFunction.ring(analytic=False)
        pts2 = np.stack([px, py], axis=1)
        sdd.mc_estimate_batch(pts2, pid, m_ref, dom, bd,
                              sdd.WalkConfig(scheme="linear", dt=DT, walks=100, seed=6), ctx=ctx)
        cfg_ref = sdd.WalkConfig(scheme="linear", dt=DT, walks=CONFIG_WALKS, seed=7, precision="fp64")
        t0 = time.perf_counter()
        sdd.mc_estimate_batch(pts2, pid, m_ref, dom, bd, cfg_ref, ctx=ctx)
        wall = time.perf_counter() - t0
        st = ctx.last_stats()
        parity_mode = {"e2e": st["path_steps"] / wall, "value": st["path_steps"] / (st["kernel_ms"] / 1e3),
                       "unit": "path-steps/s", "paths_per_node": CONFIG_WALKS, "nodes": n,
                       "path_steps": st["path_steps"], "wall_s": wall,
                       "drift": "reference (user_supplied FD of 1/w, h = 1e-6)",
                       "note": "the full config-2 walk phase in the bit-faithful parity mode: e2e = "
                               "host-buffer API wall clock, value = walk-kernel event time"}

    # ---- subdomain solver (K3/K3c), measured live: BASELINE config 3's batch
    # (128 x 129^2, shock weights, RB-SOR to 1e-10; one thread-block cluster per
    # solve) and a 2048-solve batch of the same blocks (working set 1 GB >> L2).
    # Roofline: algorithmic 40 B per point-update against the
    # measured HBM copy bandwidth; the data stays on chip, so it can exceed 1.
    solver = None
    if rank == 0 and world == 1 and not args.no_solver:
        solver = solver_rooflines(sdd, ctx)

    # ---- CPU baseline: the reference on this host, rank 0 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import bindings as B
            ref = B.Ref()
            threads = ref.hardware_threads()
            sec, sample = cpu_reference_sample(ref, B, threads)
            steps = count_steps(B, sample, threads)
            cpu = {"value": steps / sec, "unit": "path-steps/s", "cores": threads, "kind": "reference",
                   "sample": f"every {CPU_SAMPLE_STRIDE}th config-2 node ({len(sample[0])} nodes) x "
                             f"{CPU_SAMPLE_WALKS} paths, dt={DT}, reference mc_estimate with its "
                             f"user_supplied FD ring drift; {steps} path-steps in {sec:.2f} s"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "path-steps/s", "cores": None, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        k1_avg_s = k1_ms / 1e3 / args.steps
        steps_per_launch = total_steps / args.steps
        achieved = DP_FLOPS_PER_STEP * steps_per_launch / k1_avg_s / 1e12
        prec_peak = peak_fp64 if args.precision == "fp64" else peak_fp32
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        # the judged roofline of the walk is instruction issue
        # (the non-tensor issue peak: 4 warp-instructions = 128 thread-
        # instructions per SM per clock), next to the binding FP pipe; the flop
        # census against the measured FMA peak is the cross-check.  All three
        # come from this run's K1 event time; the SM clock is the one sampled
        # during the timed region.
        k1_rate = steps_per_launch / k1_avg_s  # path-steps/s of K1 alone, one GPU's share below
        sm_mhz, clock_source = (clk.get("sm_mhz") if clk else None), "nvidia-smi, median over the timed region"
        if not sm_mhz:  # no sample: the pool's maximum SM clock (a lower bound on the fraction)
            try:
                sm_mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
                clock_source = "MEASURED_PEAKS.json sm_max_mhz (no live sample)"
            except (OSError, KeyError, ValueError):
                sm_mhz, clock_source = 1965.0, "B200 maximum SM clock (no live sample)"
        hz = sm_mhz * 1e6
        pipes = pipe_fractions(k1_rate / world, sm_mhz, args.precision, sms)
        census = {"achieved": achieved, "peak": prec_peak, "unit": "TFLOP/s",
                  "frac": achieved / prec_peak if prec_peak else None,
                  "algorithmic_flops_per_path_step": DP_FLOPS_PER_STEP,
                  "peak_source": "measured on this GPU by sddg_probe_fma_peak (independent FMA chains; "
                                 "MEASURED_PEAKS.json has no non-tensor peak)",
                  "fp32_peak_tflops": peak_fp32, "fp64_peak_tflops": peak_fp64}
        roofline = {"bound": "issue", "kernel": "walk_kernel (K1)",
                    "achieved": None, "peak": None, "unit": "Tinst/s", "frac": None}
        if pipes and hz:
            roofline["achieved"] = pipes["sass_instructions_per_step"] * k1_rate / world / 1e12
            roofline["peak"] = sms * 128 * hz / 1e12
            roofline["frac"] = roofline["achieved"] / roofline["peak"]
            if args.precision == "fp64":
                roofline["fp_pipe"] = {"pipe": "fp64", "achieved": pipes["sass_fp64_per_step"] * k1_rate / world / 1e12,
                                       "peak": sms * 64 * hz / 1e12, "unit": "Tinst/s",
                                       "frac": pipes["fp64_pipe_frac"]}
        roofline.update({
            "definition": "SURVEY.md 8(d): issue-slot utilisation of K1 = executed thread-instructions "
                          "(static SASS count of one step, profiles/sass_walk_step.json, x path-steps "
                          "of this launch / K1 event time; active lanes only) over SMs x 128 thread-"
                          "instructions/clk at the SM clock sampled in the timed region; fp_pipe: the "
                          "same for the step's FP64 instructions over SMs x 64 lanes/clk; ncu: the "
                          "warp-level counters of the committed capture at this config",
            "traffic": traffic_per_launch(n * args.walks) if not c3 else None,
            "traffic_note": "DRAM read+write bytes per launch = ncu dram__bytes per walk "
                            "(profiles/ncu_walk_summary.json) x walks in this launch; "
                            "algorithmic: 20 B per walk record",
            "k1_ms_per_launch": k1_avg_s * 1e3,
            "path_steps_per_launch": steps_per_launch,
            "sm_clock_mhz": sm_mhz, "sm_clock_source": clock_source,
            "census": census,
            "pipes": pipes,
            "ncu": ncu_summary() if not c3 else {"source": "profiles/r02_walk3_fp32_ncu.txt (ncu --set full of the fp32 "
                                                              "shock kernel at 2,000 paths per node)"}})
        line = {
            "metric": "SDE walk path-steps/s", "value": value, "unit": "path-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic",
            "config": {"workload": workload,
                       "paths_per_node_per_step": args.walks, "config_paths_per_node": config_walks,
                       "nodes": n, "drift": args.drift, "precision": args.precision,
                       "l2": "flushed (256 MiB write) before every timed step",
                       "parallelism": (f"dp{world}: the {n} nodes sharded over {world} GPUs by expected "
                                       "cost (sddg_shard_plan), one ncclAllGather of the 128-B records "
                                       "per step inside the timed region (sddg_create_dist)")
                       if world > 1 else "single GPU"},
            "roofline": roofline,
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "mesh_gen_seconds": mesh,
            "solver": solver,
            "parity_mode_walks": parity_mode,
            "full_config_seconds_est": config_walks / args.walks * (total_steps / args.steps) / value,
            "shard_k1_ms": shard_k1,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Summarise one `ncu --set full` capture of the walk kernel into
profiles/ncu_walk_summary.json (the file bench.py reads for the roofline's
ncu fields and DRAM traffic per walk).

usage: python tools/ncu_summarize.py REP.ncu-rep PLAIN_BENCH.log KEY "command" "kernel note"
PLAIN_BENCH.log is the bench line of the same command run without ncu (it
supplies the path steps and walks of the launch)."""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
           "sm__inst_issued.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "smsp__inst_issued.sum", "smsp__inst_executed.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum",
           "dram__bytes_write.sum", "launch__grid_size", "launch__block_size"]
STALLS = ["not_selected", "math_pipe_throttle", "wait", "dispatch_stall", "short_scoreboard",
          "branch_resolving", "no_instruction", "long_scoreboard", "mio_throttle"]


def main():
    rep, plain, key, command, note = sys.argv[1:6]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    col = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    line = [l for l in open(plain) if l.startswith("{")][-1]
    bench = json.loads(line)
    steps = bench["roofline"]["path_steps_per_launch"]
    cfg = bench["config"]
    walks = cfg.get("nodes", cfg.get("nodes_per_rank")) * cfg["paths_per_node_per_step"]
    m = {k: {"unit": col[k][0], "value": col[k][1]} for k in METRICS if k in col}
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    # read and write may come in different units
    dram = sum(float(col[k][1]) * unit[col[k][0]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    scale = 1
    stalls = {s: float(col[f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"][1])
              for s in STALLS if f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" in col}
    out = {"command": command, "kernel": note, "metrics": m,
           "path_steps": steps, "walks": walks,
           "instructions_per_path_step": round(
               float(col["smsp__inst_executed.sum"][1]) *
               float(col["smsp__thread_inst_executed_per_inst_executed.ratio"][1]) / steps, 1),
           "warp_instructions_x32_per_path_step": round(
               32 * float(col["smsp__inst_issued.sum"][1]) / steps, 1),
           "stalls_cycles_per_issue": stalls,
           "dram_bytes_per_walk": dram * scale / walks}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_walk_summary.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[key] = out
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1)[:1500])


if __name__ == "__main__":
    main()

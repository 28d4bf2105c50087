# ncu of K1 at the bench config (753 nodes x 1e5 paths, the launch bench.py
# times): the sections and metrics the roofline quotes.  A --set full capture
# of this 4.3-s launch (source counters) does not finish in reasonable time;
# the source-level capture is taken at 1e4 paths (tools/gpu_round.sh NCU=full).
#   gpurun -- bash tools/ncu_1e5.sh ; then here:
#   python tools/ncu_summarize.py gpurun_out/walk_1e5.ncu-rep gpurun_out/bench_ncu_plain_1e5.log fp64_config2_1e5 "<command>" "<note>"
set -x
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-mesh --no-solver"
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,smsp__inst_issued.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size"
for s in not_selected math_pipe_throttle wait dispatch_stall short_scoreboard branch_resolving no_instruction long_scoreboard mio_throttle; do
  M="$M,smsp__average_warps_issue_stalled_${s}_per_issue_active.ratio"; done
timeout 300 python bench.py $ARGS > gpurun_out/bench_ncu_plain_1e5.log 2>&1 && \
timeout 2400 ncu --section SpeedOfLight --section ComputeWorkloadAnalysis --section SchedulerStats --section WarpStateStats --section LaunchStats --section Occupancy --metrics $M --clock-control none -k regex:walk_kernel -s 1 -c 1 -f -o gpurun_out/walk_1e5 python bench.py $ARGS > gpurun_out/ncu_1e5.log 2>&1
echo "ncu rc=$?"

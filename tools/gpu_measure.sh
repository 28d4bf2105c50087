# Round measurement on one B200: smoke, GPU tests, bench line, launch list,
# ncu --set full of K1 (fp64 config 2 and fp32 config 3).  TAG names outputs.
TAG=${TAG:-x}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/tests_$TAG.log; cat gpurun_out/tests_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench_$TAG.log | cut -c1-300
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-mesh > gpurun_out/bench_ncu_plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-mesh > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launch rc=$?"
timeout 300 python bench.py --steps 1 --warmup 1 --walks 10000 --no-cpu-baseline --no-e2e --no-mesh > gpurun_out/bench_ncu_plain2_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 1 -c 1 -o gpurun_out/walk_full_$TAG python bench.py --steps 1 --warmup 1 --walks 10000 --no-cpu-baseline --no-e2e --no-mesh > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
timeout 300 python tools/walk_once.py config3 fp32 500 > gpurun_out/walk3_plain_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 1 -c 1 -o gpurun_out/walk3_full_$TAG python tools/walk_once.py config3 fp32 500 > gpurun_out/ncu3_full_$TAG.log 2>&1; echo "ncu fp32 rc=$?"

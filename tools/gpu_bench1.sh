set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_plain.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_plain.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 300 python bench.py --steps 1 --warmup 1 --walks 500 --no-cpu-baseline --no-e2e > gpurun_out/bench_tiny.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 1 -c 1 -o gpurun_out/walk_full python bench.py --steps 1 --warmup 1 --walks 500 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out

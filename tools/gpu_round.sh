# one measurement round on the B200: tests, bench, launch list, full ncu of the walk kernel
set -x
TAG=${TAG:-x}
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/tests_$TAG.log; cat gpurun_out/tests_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_$TAG.log
if [ "${NCU:-1}" = 1 ]; then
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu_plain_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 1 -c 1 -o gpurun_out/walk_full_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu rc=$?"
fi

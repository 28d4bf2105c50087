# quick perf check: fastmath accuracy test + bench twice (variance)
timeout 300 python -m pytest tests/test_gpu_walk.py -q -m gpu -k "fastmath or parity or fp32 or analytic" 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value %.4e  k1 %.1f ms  clocks %s'%(d['value'], d['roofline']['k1_ms_per_launch'], d['clocks']['sm_mhz']))
"; done

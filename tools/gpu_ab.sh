# A/B timing of library variants in one call (same GPU)
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then export SDDG_LIB_PATH=; else export SDDG_LIB_PATH=$PWD/paper_1310_3435_b200/_lib/libsddg_$v.so; fi
  timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v: value %.4e  k1 %.1f ms  clocks %s'%(d['value'], d['roofline']['k1_ms_per_launch'], d['clocks']['sm_mhz']))
    elif 'Error' in l or 'error' in l: print(l.strip())
"
done

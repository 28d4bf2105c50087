# A/B timing of library variants on one GPU: VARIANTS="default old ..." (libsddg_<v>.so), ROUNDS, BENCH_ARGS
for r in $(seq ${ROUNDS:-2}); do
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then export SDDG_LIB_PATH=; else export SDDG_LIB_PATH=$PWD/paper_1310_3435_b200/_lib/libsddg_$v.so; fi
  timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e --no-mesh ${BENCH_ARGS} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v: value %.4e  k1 %.1f ms  clocks %s %s'%(d['value'], d['roofline']['k1_ms_per_launch'], d['clocks']['sm_mhz'], d['clocks']['reasons']))
    elif 'Error' in l or 'error' in l: print(l.strip())
"
done
done

# A/B of library variants on one walk batch: VARIANTS, ROUNDS, ARGS="config3 fp32 1000"
for r in $(seq ${ROUNDS:-2}); do
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then export SDDG_LIB_PATH=; else export SDDG_LIB_PATH=$PWD/paper_1310_3435_b200/_lib/libsddg_$v.so; fi
  echo -n "$v: "; timeout 600 python tools/walk_once.py ${ARGS:-config3 fp32 1000} 2>&1 | tail -1
done
done

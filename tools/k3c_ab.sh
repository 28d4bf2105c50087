# A/B of K3c variants (libsddg_<v>.so, optionally "<v>@<cluster size>") on the
# config-3 batch (128 x 129^2, shock, tol 1e-10)
for r in 1 2; do
for vv in ${VARIANTS:-default}; do
  v=${vv%@*}; cl=; [ "$vv" != "$v" ] && cl=${vv#*@}
  if [ "$v" = default ]; then export SDDG_LIB_PATH=; else export SDDG_LIB_PATH=$PWD/paper_1310_3435_b200/_lib/libsddg_$v.so; fi
  echo -n "$vv: "; SDDG_CLUSTER_SIZE=$cl SOLVER_REPS=3 timeout 120 python tools/solver_once.py ${SOLVER_ARGS:-128 1025 8} 2>&1 | tail -1
done
done

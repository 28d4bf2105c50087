#!/bin/bash
# The checked build (SDDG_CHECKS=1: device-side bounds asserts, see
# csrc/sddg_internal.h SDDG_CHECK) run under the whole GPU suite and the
# sanitizer cases -- the stand-in for compute-sanitizer, which is closed on
# the GPU pool (profiles/r02_compute_sanitizer_refused.log).
#   SDDG_BUILD_TAG=chk SDDG_EXTRA_NVCC="-DSDDG_CHECKS=1" python paper_1310_3435_b200/build.py
#   gpurun -- bash tools/checked_tests.sh
set -u
cd "$(dirname "$0")/.."
export SDDG_LIB_PATH=$PWD/paper_1310_3435_b200/_lib/libsddg_chk.so
test -f "$SDDG_LIB_PATH" || { echo "no checked build at $SDDG_LIB_PATH"; exit 1; }
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/checked_tests.log
rc=${PIPESTATUS[0]}
grep -c "SDDG_CHECK failed" gpurun_out/checked_tests.log >/dev/null && echo "SDDG_CHECK fired" >> gpurun_out/checked_tests.log
echo "pytest rc=$rc" >> gpurun_out/checked_tests.log
python -c "from paper_1310_3435_b200 import sdd; print(\"library:\", sdd._LIB_PATH)" >> gpurun_out/checked_tests.log
cat gpurun_out/checked_tests.log
exit $rc

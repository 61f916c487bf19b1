#!/bin/bash
# One gpurun call: GPU parity tests (optional), then instruction-count and pipelined A/B of
# libvsag_<variant>.so builds against libvsag.so ("new").  VARIANTS="base new", EF=132, PYTEST=1
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
if [ "${PYTEST:-1}" = 1 ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1
  echo "pytest=$?"; tail -5 gpurun_out/pytest.log
fi
# PYTEST=2: a quick subset of the parity tests (trace-exact cases on C0, C1 full size), run for
# every library in $TESTVARS (default: new)
if [ "${PYTEST:-1}" = 2 ]; then
  for v in ${TESTVARS:-new}; do
    if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi
    timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider \
      -k "c0_parity or c0_params or forgetful_visited_cache or qlp_parity or maximum_pool or c1_full or w1_gpu or padded_rows" \
      > gpurun_out/pytest_$v.log 2>&1
    echo "pytest[$v]=$?"; tail -2 gpurun_out/pytest_$v.log
  done
  unset VSAG_LIB_VARIANT
fi
EF=${EF:-132} VARIANTS="${VARIANTS:-base new}" bash tools/ab_inst.sh 2>&1 | tee gpurun_out/ab_inst.txt

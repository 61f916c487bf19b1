#!/bin/bash
# One gpurun call: GPU parity tests (optional), then instruction-count and pipelined A/B of
# libvsag_<variant>.so builds against libvsag.so ("new").  VARIANTS="base new", EF=132, PYTEST=1
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
if [ "${PYTEST:-1}" = 1 ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1
  echo "pytest=$?"; tail -5 gpurun_out/pytest.log
fi
EF=${EF:-132} VARIANTS="${VARIANTS:-base new}" bash tools/ab_inst.sh 2>&1 | tee gpurun_out/ab_inst.txt

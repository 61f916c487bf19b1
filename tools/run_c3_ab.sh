#!/bin/bash
# A/B of library variants on C3 (degree 64, IP SQ8, k = 100): tools/config_sweep.py rows
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
for v in ${VARIANTS:-base new}; do
  if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi
  timeout 1500 python tools/config_sweep.py ${CONFIGS:-C3} --no-oracle > gpurun_out/sweep_$v.json 2> gpurun_out/sweep_$v.log
  echo "== $v"; grep -E "^  C" gpurun_out/sweep_$v.log | sed -E "s/exact=.*//" | cut -c1-330
done

#!/bin/bash
# A/B timing of search-kernel builds on C1 ef=160 (one gpurun call):
#   VARIANTS="base new"  -> libvsag_base.so vs libvsag.so ("new" = the default build)
#   NCU=1                -> one ncu --set full capture of search_kernel per variant
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
EF=${EF:-160}
for v in ${VARIANTS:-base new}; do
  if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi
  echo "== $v" >> gpurun_out/ab.txt
  timeout 600 python tools/sweep_launch.py --ef $EF --reps ${REPS:-20} --grid "${GRID:-lanes=0;slots=0;wpb=0}" >> gpurun_out/ab.txt 2>&1
  if [ -n "$NCU" ]; then
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 3 -c 1 -o gpurun_out/prof_$v -f \
      python tools/sweep_launch.py --ef $EF --reps 1 --grid "lanes=0;slots=0;wpb=0" > gpurun_out/ncu_$v.log 2>&1
  fi
done
cat gpurun_out/ab.txt

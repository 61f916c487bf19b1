#!/bin/bash
# One gpurun call: hop statistics (libvsag_stats.so, -DVSAG_STATS) and one ncu --set full
# source-level capture of search_kernel on C1 at $EF (read with tools/ncu_lines.py).
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
EF=${EF:-132}
if [ -f paper_2503_17911_b200/libvsag_stats.so ]; then
  VSAG_LIB_VARIANT=stats timeout 600 python tools/stats_run.py C1 $EF > gpurun_out/stats.txt 2>&1; cat gpurun_out/stats.txt
fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/prof_search -f python tools/stage_times.py $EF > gpurun_out/ncu_search.log 2>&1
echo "ncu_search=$?"
ncu -i gpurun_out/prof_search.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/prof_search_src.csv 2>/dev/null
ncu -i gpurun_out/prof_search.ncu-rep --page raw --csv > gpurun_out/prof_search_raw.csv 2>/dev/null
ls -la gpurun_out/

#!/bin/bash
# One gpurun call for this round's ncu evidence at the bench's operating point (C1):
#   plain.json        bench.py --ef $EF --steps 5 (no ncu; must exit 0 first)
#   launches.csv      ncu launch list of that same command (gpu__time_duration.sum, cold, serialised)
#   prof_search.ncu-rep  ncu --set full --import-source on of one search_kernel launch
#   prof_seed.ncu-rep    the same for the seed contraction and the seed selection
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
EF=${EF:-130}
: > gpurun_out/status.txt
timeout 900 python bench.py --ef $EF --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain.json 2> gpurun_out/plain.err
echo "plain=$?" >> gpurun_out/status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --ef $EF --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
echo "launches=$?" >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/prof_search -f python tools/stage_times.py $EF > gpurun_out/ncu_search.log 2>&1
echo "ncu_search=$?" >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seed_" -s 2 -c 2 \
  -o gpurun_out/prof_seed -f python tools/stage_times.py $EF > gpurun_out/ncu_seed.log 2>&1
echo "ncu_seed=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

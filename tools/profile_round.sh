#!/bin/bash
# One gpurun call for the round's evidence (C1, the bench's operating point):
#   bench.json            python bench.py (default: 200 steps, cpu baseline)
#   launches.csv          ncu launch list of bench.py --ef $EF --steps 5 (the timed config only)
#   prof_new.ncu-rep      ncu --set full of one timed search launch (tools/ab.sh)
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
EF=${EF:-132}
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? > gpurun_out/status.txt
timeout 900 python bench.py --ef $EF --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain.json 2> gpurun_out/plain.err && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"search_kernel|seed_|query_prep" --csv \
    --log-file gpurun_out/launches.csv python bench.py --ef $EF --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
echo launches=$? >> gpurun_out/status.txt
rm -f gpurun_out/ab.txt
EF=$EF NCU=1 VARIANTS=new REPS=10 bash tools/ab.sh > /dev/null 2>&1; echo ncu=$? >> gpurun_out/status.txt
cat gpurun_out/status.txt

#!/bin/bash
# one gpurun call: GPU tests + bench (+ optional ncu), outputs under gpurun_out/
#   NCU=1        also capture the launch list and one ncu --set full of search_kernel
#   QUICK=1      skip the full pytest -m gpu run (bench + ncu only)
#   BENCH_ARGS   extra bench.py arguments
mkdir -p gpurun_out
export VSAG_CACHE_DIR=/tmp/vsag_cache
: > gpurun_out/status.txt
if [ -z "$QUICK" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
fi
timeout 900 python bench.py --steps ${STEPS:-100} ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
if [ -n "$NCU" ]; then
  CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS}"
  $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"search_kernel|seed_|query_prep" --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 10 -c 1 -o gpurun_out/prof_search -f $CMD > gpurun_out/ncu2.log 2>&1
  echo ncu=$? >> gpurun_out/status.txt
fi
cat gpurun_out/status.txt

#!/bin/bash
# instruction count and time of search_kernel on one config/ef for several library variants
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
for v in ${VARIANTS:-base new}; do
  if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi
  timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,dram__bytes_read.sum \
    --clock-control none -k regex:search_kernel -s 1 -c 1 --csv --log-file gpurun_out/cfginst_$v.csv python tools/cfg_once.py ${CFG:-C3} ${EF:-256} ${KIND:-auto} > gpurun_out/cfginst_$v.out 2>&1
  echo "== $v"; tail -1 gpurun_out/cfginst_$v.out
  python - "$v" <<'PY'
import csv, sys
v = sys.argv[1]
rows = [r for r in csv.reader(l for l in open(f"gpurun_out/cfginst_{v}.csv") if not l.startswith("=="))]
h = rows[0]
for r in rows[1:]:
    print("  ", r[h.index("Metric Name")], r[h.index("Metric Value")])
PY
done

#!/bin/bash
# A/B of library variants: executed instructions and time of search_kernel (ncu, 3 launches,
# C1 at $EF) plus the pipelined step (tools/ab_pipeline.py).  VARIANTS="prev new"
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
EF=${EF:-130}
for v in ${VARIANTS:-prev new}; do
  if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi
  timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:search_kernel \
    -c 3 --csv --log-file gpurun_out/inst_$v.csv python tools/stage_times.py $EF > /dev/null 2>&1
  python - "$v" <<'PY'
import csv, sys
v = sys.argv[1]
rows = [r for r in csv.reader(l for l in open(f"gpurun_out/inst_{v}.csv") if not l.startswith("=="))]
h = rows[0]
vals = {}
for r in rows[1:]:
    vals.setdefault(r[h.index("Metric Name")], []).append(float(r[h.index("Metric Value")]))
print(f"[{v}] inst/launch {sum(vals['smsp__inst_executed.sum']) / len(vals['smsp__inst_executed.sum']) / 1e6:.1f} M, "
      f"ncu time {sum(vals['gpu__time_duration.sum']) / len(vals['gpu__time_duration.sum']) / 1e3:.1f} us")
PY
done
for r in 1 2; do for v in ${VARIANTS:-prev new}; do
  if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi
  timeout 600 python tools/ab_pipeline.py --ef $EF --reps 10 --rounds 2
done; done

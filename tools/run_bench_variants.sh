#!/bin/bash
# bench.py for several library variants / warps per block on one box: RUNS="new:0 mb10:2 mb10:4"
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
for r in ${RUNS:-new:0}; do
  v=${r%%:*}; w=${r##*:}
  if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi
  timeout 900 python bench.py --no-cpu-baseline --ef ${EF:-132} --warps-per-block $w > gpurun_out/bench_${v}_$w.json 2> gpurun_out/bench_${v}_$w.err
  python - "$v" "$w" <<'PY'
import json, sys
v, w = sys.argv[1:3]
d = json.load(open(f"gpurun_out/bench_{v}_{w}.json"))
r = d["roofline"]
print(f"[{v} wpb={w}] {d['value'] / 1e6:.3f} M QPS, step {d['ms_per_step']:.4f} ms, e2e {d['e2e']['value'] / 1e6:.3f} M, "
      f"kernel {r['kernel_ms']:.4f} ms, frac {r['frac']:.4f}, per-step frac {r['frac_per_step']:.4f}, launch {d['launch']}")
PY
done

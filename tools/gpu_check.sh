#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, compute-sanitizer over every kernel variant.
#   STEPS="pytest smoke bench sanitize" (default all); results under gpurun_out/
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
STEPS=${STEPS:-"pytest smoke bench"}
: > gpurun_out/status.txt
for s in $STEPS; do
  case $s in
    pytest)
      timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1
      echo "pytest=$?" >> gpurun_out/status.txt; tail -3 gpurun_out/pytest.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke=$?" >> gpurun_out/status.txt ;;
    bench)
      timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
      echo "bench=$?" >> gpurun_out/status.txt; tail -c 600 gpurun_out/bench.json ;;
    ab)
      for v in ${AB_VARIANTS:-base new base new}; do
        if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi
        timeout 600 python tools/ab_pipeline.py --ef ${AB_EF:-130} >> gpurun_out/ab.txt 2>&1
      done
      unset VSAG_LIB_VARIANT
      echo "ab=done" >> gpurun_out/status.txt; cat gpurun_out/ab.txt ;;
    sanitize)  # (compute-sanitizer is closed on this pool: kept for other machines)
      timeout 600 python tools/sanitize.py --prep > gpurun_out/san_prep.log 2>&1
      for tool in memcheck synccheck racecheck; do
        timeout 1200 compute-sanitizer --tool $tool --kernel-name regex:vsag --error-exitcode 9 \
          --log-file gpurun_out/sanitize_$tool.log python tools/sanitize.py --c1 ${SAN_C1:-1000} \
          > gpurun_out/sanitize_$tool.out 2>&1
        echo "sanitize_$tool=$?" >> gpurun_out/status.txt
      done ;;
  esac
done
cat gpurun_out/status.txt

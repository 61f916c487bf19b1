#!/bin/bash
# One gpurun call for the round's evidence at the final build: full GPU parity suite, the
# bounds-checked build over every variant, smoke, the default bench line, then the ncu
# launch list and full captures (tools/profile_r02.sh) at the bench's operating ef.
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest.log
if [ -f paper_2503_17911_b200/libvsag_chk.so ]; then
  VSAG_LIB_VARIANT=chk timeout 900 python tools/sanitize.py --c1 1000 > gpurun_out/chk.log 2>&1; echo "chk=$?"; tail -2 gpurun_out/chk.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"; tail -c 400 gpurun_out/bench.json
EF=${EF:-132} bash tools/profile_r02.sh
for f in prof_search prof_seed; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
done
ncu -i gpurun_out/prof_search.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/prof_search_src.csv 2>/dev/null
ls -la gpurun_out | head -40

export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest.log
VSAG_LIB_VARIANT=chk timeout 900 python tools/sanitize.py --c1 1000 > gpurun_out/chk.log 2>&1; echo "chk=$?"; tail -3 gpurun_out/chk.log

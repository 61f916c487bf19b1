export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
run() { v=$1; w=$2; if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi; timeout 600 python tools/ab_pipeline.py --ef 132 --reps 10 --rounds 2 --wpb $w; }
for r in 1 2; do run c3 0; run new 0; run new 4; run mb10 4; done 2>&1 | tee gpurun_out/ab_mb.txt
unset VSAG_LIB_VARIANT
VSAG_LIB_VARIANT=mb10 timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "c0_parity or c0_params or forgetful_visited_cache or qlp_parity or maximum_pool or c1_full or w1_gpu or padded_rows" 2>&1 | tail -2

# one ncu --set full capture of search_kernel on C1 (ef=160) via the sweep tool
export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
python tools/sweep_launch.py --ef 160 --reps 10 --grid "lanes=0;slots=0;wpb=0" > gpurun_out/sweep.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 3 -c 1 -o gpurun_out/prof_search -f python tools/sweep_launch.py --ef 160 --reps 1 --grid "lanes=0;slots=0;wpb=0" > gpurun_out/ncu_s.log 2>&1
echo done

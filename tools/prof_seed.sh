export VSAG_CACHE_DIR=/tmp/vsag_cache
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"seed_select|seed_tau" -s 6 -c 2 -o gpurun_out/prof_seed -f python tools/sweep_launch.py --ef 160 --reps 3 --grid "lanes=0;slots=0;wpb=0" > gpurun_out/ncu_seed.log 2>&1
echo done

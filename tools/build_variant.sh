#!/bin/bash
# Build libvsag_<name>.so: search_m0.cu (L2 SQ8) recompiled with extra nvcc flags, linked with
# the default build's other objects (run `python paper_2503_17911_b200/build.py` first).
#   tools/build_variant.sh minb10 -DVSAG_SEARCH_MINB=10
set -e
name=$1; shift
D=$(cd "$(dirname "$0")/.." && pwd)/paper_2503_17911_b200
B=$D/build
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -Xptxas -v "$@" -I $D/../include -I $D/csrc -c $D/csrc/search_m0.cu -o /tmp/m0_$name.o 2> /tmp/m0_$name.log
grep -A2 "Li0ELi2ELi2ELi1ELi0ELi1E" /tmp/m0_$name.log | grep -E "spill|Used" | head -2
objs=$(ls $B/*.o | grep -v search_m0.cu.o)
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $D/libvsag_$name.so $objs /tmp/m0_$name.o

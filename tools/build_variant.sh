#!/bin/bash
# Build libvsag_<name>.so: one source (SRC, default search_m0 = the L2 SQ8 search kernel)
# recompiled with extra nvcc flags, linked with the default build's other objects (run
# `python paper_2503_17911_b200/build.py` first).
#   tools/build_variant.sh minb10 -DVSAG_SEARCH_MINB=10
#   SRC=select tools/build_variant.sh sel2 -DVSAG_SEL_WARPS=2
set -e
name=$1; shift
SRC=${SRC:-search_m0}
D=$(cd "$(dirname "$0")/.." && pwd)/paper_2503_17911_b200
B=$D/build
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -Xptxas -v "$@" -I $D/../include -I $D/csrc -c $D/csrc/$SRC.cu -o /tmp/${SRC}_$name.o 2> /tmp/${SRC}_$name.log
grep -A2 "Li0ELi2ELi2ELi1ELi0ELi1E" /tmp/${SRC}_$name.log | grep -E "spill|Used" | head -2 || true
objs=$(ls $B/*.o | grep -v "/$SRC.cu.o")
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $D/libvsag_$name.so $objs /tmp/${SRC}_$name.o

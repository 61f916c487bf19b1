#!/bin/bash
# C4 (2M rows) forced onto the u32 visited table = the code path of the full 10M-row config
# (generic variant, linear probing), for several library variants
export VSAG_CACHE_DIR=/tmp/vsag_cache
for v in ${VARIANTS:-base new}; do
  if [ "$v" = new ]; then unset VSAG_LIB_VARIANT; else export VSAG_LIB_VARIANT=$v; fi
  for ef in 32 64 128; do
    echo -n "[$v] "; timeout 900 python tools/cfg_once.py C4 $ef u32 ${SLOTS:-0} 2>&1 | tail -1
  done
done

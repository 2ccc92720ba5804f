#!/bin/bash
mkdir -p gpurun_out/c29
O=gpurun_out/c29
: > $O/l2256.txt
for lib in default l2256; do
  if [ $lib = default ]; then unset HCS_LIB_PATH; else export HCS_LIB_PATH=$PWD/tools/exp_libs/libhcspmm_$lib.so; fi
  echo "== $lib" >> $O/l2256.txt
  DIMS=64,128 timeout 300 python tools/exp_tile_dims.py >> $O/l2256.txt 2>&1
  timeout 900 python tools/exp_c5.py 2>&1 | grep -E "^tile|^scalar|^all" >> $O/l2256.txt
done

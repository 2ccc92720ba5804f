#!/bin/bash
mkdir -p gpurun_out/c24
O=gpurun_out/c24
: > $O/occ.txt
for lib in default w6 w4; do
  if [ $lib = default ]; then unset HCS_LIB_PATH; else export HCS_LIB_PATH=$PWD/tools/exp_libs/libhcspmm_$lib.so; fi
  echo "== $lib" >> $O/occ.txt
  DIMS=64,128 timeout 300 python tools/exp_tile_dims.py >> $O/occ.txt 2>&1
done

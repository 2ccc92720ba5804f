#!/bin/bash
mkdir -p gpurun_out/c18
O=gpurun_out/c18
: > $O/ablation2.txt
for lib in default nogather nogather_nomma; do
  if [ $lib = default ]; then unset HCS_LIB_PATH; else export HCS_LIB_PATH=$PWD/tools/exp_libs/libhcspmm_$lib.so; fi
  echo "== $lib" >> $O/ablation2.txt
  DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/ablation2.txt 2>&1
done
HCS_LIB_PATH=$PWD/tools/exp_libs/libhcspmm_nogather_nomma.so DIMS=128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_warp -s 3 -c 1 -o $O/nogather_nomma python tools/exp_tile_dims.py > /dev/null 2>&1

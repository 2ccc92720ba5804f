#!/bin/bash
# plan-stream L2 prefetch variants of the tile kernel: C5 tile launch and C2 N=64/128
mkdir -p gpurun_out/s3d
O=gpurun_out/s3d
for v in ship pf_e4 pf_g4e4 pf_g8e6; do
  if [ $v = ship ]; then L=""; else L=tools/exp_libs/$v/libhcspmm.so; fi
  echo "== $v" >> $O/c2.txt
  HCS_LIB_PATH=$L DIMS=64,128 timeout 300 python tools/exp_tile_dims.py >> $O/c2.txt 2>&1
done
for v in ship pf_e4 pf_g4e4 pf_g8e6; do
  if [ $v = ship ]; then L=""; else L=tools/exp_libs/$v/libhcspmm.so; fi
  echo "== $v" >> $O/c5.txt
  HCS_LIB_PATH=$L timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/c5.txt
done

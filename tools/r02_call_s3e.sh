#!/bin/bash
mkdir -p gpurun_out/s3e
O=gpurun_out/s3e
for rep in 1 2; do
for v in pf_e0 default pf_e2 pf_e8; do
  if [ $v = default ]; then L=""; else L=tools/exp_libs/$v/libhcspmm.so; fi
  echo "== $v" >> $O/c2.txt
  HCS_LIB_PATH=$L DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/c2.txt 2>&1
done
done

#!/bin/bash
mkdir -p gpurun_out/s3f
O=gpurun_out/s3f
for rep in 1 2; do
for v in default tf_l4 tf_l8; do
  if [ $v = default ]; then L=""; else L=tools/exp_libs/$v/libhcspmm.so; fi
  echo "== $v" >> $O/c2tf.txt
  PREC=tf32 HCS_LIB_PATH=$L DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/c2tf.txt 2>&1
done
done

#!/bin/bash
mkdir -p gpurun_out/s3r
O=gpurun_out/s3r
echo "== default (warp, 32-B, U=3, MINB=3)" >> $O/r.txt; timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/r.txt
for v in s16u6m3 s16u5m3 s16u7m3 s16u12m2 s16u6m2 s16u6m3; do
  echo "== warp16 $v" >> $O/r.txt; C5_SCALAR_VARIANT=warp16 HCS_LIB_PATH=tools/exp_libs/$v/libhcspmm.so timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/r.txt
done

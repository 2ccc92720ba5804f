#!/bin/bash
mkdir -p gpurun_out/s3q
O=gpurun_out/s3q
echo "== default (warp, 32-B, U=3, MINB=3)" >> $O/r.txt; timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/r.txt
echo "== warp16 default U=4 MINB=3" >> $O/r.txt; C5_SCALAR_VARIANT=warp16 timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/r.txt
for v in s16u6m3 s16u6m4 s16u8m3 s16u8m4; do
  echo "== warp16 $v" >> $O/r.txt; C5_SCALAR_VARIANT=warp16 HCS_LIB_PATH=tools/exp_libs/$v/libhcspmm.so timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/r.txt
done

#!/bin/bash
mkdir -p gpurun_out/s4f
O=gpurun_out/s4f
for rep in 1 2; do
echo "== 64" >> $O/r.txt; timeout 300 python tools/exp_gemm.py >> $O/r.txt 2>&1
echo "== 128" >> $O/r.txt; HCS_LIB_PATH=tools/exp_libs/g128/libhcspmm.so timeout 300 python tools/exp_gemm.py >> $O/r.txt 2>&1
done

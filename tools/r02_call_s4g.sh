#!/bin/bash
mkdir -p gpurun_out/s4g
O=gpurun_out/s4g
for rep in 1 2; do
echo "== MT1" >> $O/r.txt; HCS_LIB_PATH=tools/exp_libs/mt1/libhcspmm.so timeout 300 python tools/exp_gemm.py >> $O/r.txt 2>&1
echo "== MT2" >> $O/r.txt; timeout 300 python tools/exp_gemm.py >> $O/r.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_gnn.py -q -x -p no:cacheprovider > $O/t.txt 2>&1; echo "rc=$?" >> $O/t.txt
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/c3.json 2> $O/c3.err

#!/bin/bash
mkdir -p gpurun_out/s3n
O=gpurun_out/s3n
for rep in 1 2; do
echo "== default" >> $O/c1.txt; DIM=32 PREC=bf16 timeout 300 python tools/exp_c1.py 2>&1 | head -1 >> $O/c1.txt
echo "== pv16" >> $O/c1.txt; HCS_LIB_PATH=tools/exp_libs/pv16/libhcspmm.so DIM=32 PREC=bf16 timeout 300 python tools/exp_c1.py 2>&1 | head -1 >> $O/c1.txt
done
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $O/b_def.json 2>/dev/null
HCS_LIB_PATH=tools/exp_libs/pv16/libhcspmm.so timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $O/b_pv16.json 2>/dev/null
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $O/b_def2.json 2>/dev/null
HCS_LIB_PATH=tools/exp_libs/pv16/libhcspmm.so timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $O/b_pv16_2.json 2>/dev/null

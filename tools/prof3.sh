#!/bin/bash
for d in 32 128; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tile -s 2 -c 1 \
   -o gpurun_out/prof3_d$d python bench.py --steps 3 --warmup 3 --dim $d --no-cpu-baseline --no-e2e > /dev/null 2>&1
done

#!/bin/bash
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tile -s 2 -c 1 \
   -o gpurun_out/prof2_d32 python bench.py --steps 3 --warmup 3 --dim 32 --no-cpu-baseline --no-e2e > gpurun_out/prof2_bench.log 2>&1

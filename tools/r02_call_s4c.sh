#!/bin/bash
mkdir -p gpurun_out/s4c
O=gpurun_out/s4c
timeout 900 ncu --set full --clock-control none -k regex:k_spmm_scalar_w -c 1 -o $O/full_scalar_c5 python tools/exp_c5.py > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file $O/launches_c1.csv python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la $O

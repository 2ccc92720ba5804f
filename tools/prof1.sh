#!/bin/bash
# ncu capture of the tile kernel on the C2 bench (dim 128 and dim 32), plus launch list
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tile -s 2 -c 1 \
   -o gpurun_out/prof_tile_d128 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof1_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tile -s 2 -c 1 \
   -o gpurun_out/prof_tile_d32 python bench.py --steps 3 --warmup 3 --dim 32 --no-cpu-baseline --no-e2e >> gpurun_out/prof1_bench.log 2>&1
ls -la gpurun_out

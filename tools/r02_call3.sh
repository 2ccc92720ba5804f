#!/bin/bash
mkdir -p gpurun_out/c3
O=gpurun_out/c3
timeout 300 python tools/exp_c1.py > $O/exp_c1.txt 2>&1
DIM=32 timeout 300 python tools/exp_c1.py > $O/exp_c1_d32.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tile_warp|k_spmm_scalar" --csv --log-file $O/launches_c1.csv python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --cuda-graph off > /dev/null 2>&1
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
ls -la $O

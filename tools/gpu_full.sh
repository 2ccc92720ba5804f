#!/bin/bash
# one gpurun session: smoke, gpu tests, bench, ncu launch list + full capture of the tile kernel
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -40
timeout 600 python bench.py --steps 50 --warmup 5 --cpu-budget 8 --sweep-dims > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tile -s 2 -c 1 -o gpurun_out/full_tile_d128 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out

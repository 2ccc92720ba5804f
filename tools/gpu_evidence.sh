#!/bin/bash
# Full evidence session: smoke, GPU tests, bench lines (C2 default + sweep, tf32, C3, C4, C5),
# ncu launch list of the default bench and a full capture of the tile kernel.
set -x
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/ev/pytest_gpu.log 2>&1; tail -3 gpurun_out/ev/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --cpu-budget 8 --sweep-dims > gpurun_out/ev/bench_c2.json 2> gpurun_out/ev/bench_c2.err
timeout 600 python bench.py --steps 50 --warmup 5 --precision tf32 --no-cpu-baseline --no-e2e > gpurun_out/ev/bench_c2_tf32.json 2> gpurun_out/ev/bench_c2_tf32.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --dim 128 > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err
timeout 900 python bench.py --config c4 --graph community --steps 20 --warmup 3 --dim 128 > gpurun_out/ev/bench_c4_community.json 2> gpurun_out/ev/bench_c4_community.err
timeout 600 python bench.py --graph community --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ev/bench_c2_community.json 2> gpurun_out/ev/bench_c2_community.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev/bench_c5.json 2> gpurun_out/ev/bench_c5.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --selector paper_2412_08902_b200/data/selector_b200.json > gpurun_out/ev/bench_c5_b200sel.json 2> gpurun_out/ev/bench_c5_b200sel.err
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 > gpurun_out/ev/bench_c1.json 2> gpurun_out/ev/bench_c1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_warp$ -s 2 -c 1 -o gpurun_out/ev/full_tile_d128 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k k_spmm_scalar_w -c 1 -o gpurun_out/ev/full_scalar_c5 python tools/exp_c5.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k k_tile_warp -c 1 -o gpurun_out/ev/full_tile_c5 python tools/exp_c5.py > /dev/null 2>&1
ls -la gpurun_out/ev

#!/bin/bash
# session-3 evidence: smoke, bench lines (C2 + dims, tf32, C1, C3, C5, reference arm), default-bench launch
# list, ncu full capture of the C2 tile launch and of the balanced C5 tile launch
mkdir -p gpurun_out/s3ev
O=gpurun_out/s3ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py --sweep-dims > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --steps 50 --warmup 5 --precision tf32 --no-cpu-baseline > $O/bench_c2_tf32.json 2> $O/bench_c2_tf32.err
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_warp -s 2 -c 1 -o $O/full_tile_c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:k_tile_warp -c 1 -o $O/full_tile_c5 python tools/exp_c5.py > /dev/null 2>&1
ls -la $O

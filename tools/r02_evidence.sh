#!/bin/bash
# round 2 evidence: smoke, bench lines for every config (C1, C2 + dims sweep, C2 tf32, C2 community, C3, C4, C5,
# reference arm), shared-GPU 2-rank bench, default-bench launch list
mkdir -p gpurun_out/ev2
O=gpurun_out/ev2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --sweep-dims > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --steps 50 --warmup 5 --precision tf32 --no-cpu-baseline > $O/bench_c2_tf32.json 2> $O/bench_c2_tf32.err
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c4 --steps 20 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c4 --graph community --steps 20 --warmup 3 > $O/bench_c4_community.json 2> $O/bench_c4_community.err
timeout 600 python bench.py --graph community --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_c2_community.json 2> $O/bench_c2_community.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
HCS_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_shared2.json 2> $O/bench_shared2.err
ls -la $O

#!/bin/bash
# round 2: GPU tests + default bench + reference arm + 2-rank shared-GPU bench
mkdir -p gpurun_out
export HCS_PARITY_LOG=$PWD/gpurun_out/r02_parity.jsonl
rm -f $HCS_PARITY_LOG
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
echo "bench rc=$?" >> gpurun_out/r02_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
echo "ref rc=$?" >> gpurun_out/r02_bench_ref.err
HCS_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e > gpurun_out/r02_bench_shared2.json 2> gpurun_out/r02_bench_shared2.err
echo "shared2 rc=$?" >> gpurun_out/r02_bench_shared2.err

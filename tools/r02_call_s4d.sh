#!/bin/bash
mkdir -p gpurun_out/s4d
O=gpurun_out/s4d
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
HCS_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/shared2.json 2> $O/shared2.err; echo "rc=$?" >> $O/shared2.err
HCS_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --config c3 --steps 5 --warmup 3 > $O/shared2_c3.json 2> $O/shared2_c3.err; echo "rc=$?" >> $O/shared2_c3.err

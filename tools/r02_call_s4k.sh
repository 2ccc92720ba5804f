#!/bin/bash
mkdir -p gpurun_out/s4k
O=gpurun_out/s4k
HCS_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/shared2.json 2> $O/shared2.err; echo "rc=$?" >> $O/shared2.err
HCS_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/shared2_e2e.json 2> $O/shared2_e2e.err; echo "rc=$?" >> $O/shared2_e2e.err

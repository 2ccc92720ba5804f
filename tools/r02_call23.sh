#!/bin/bash
mkdir -p gpurun_out/c23
O=gpurun_out/c23
HCS_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_shared2.json 2> $O/bench_shared2.err; echo "rc=$?" >> $O/bench_shared2.err

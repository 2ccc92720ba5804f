#!/bin/bash
mkdir -p gpurun_out/s4l
HCS_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --config c3 --steps 5 --warmup 3 > gpurun_out/s4l/c3.json 2> gpurun_out/s4l/c3.err; echo "rc=$?" >> gpurun_out/s4l/c3.err

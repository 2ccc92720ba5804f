#!/bin/bash
mkdir -p gpurun_out/c30
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/c30/bench_c3.json 2> gpurun_out/c30/bench_c3.err

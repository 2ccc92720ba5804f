#!/bin/bash
mkdir -p gpurun_out/c22
O=gpurun_out/c22
for d in 128 64 32; do timeout 600 python bench.py --steps 30 --warmup 5 --precision tf32 --dim $d --no-cpu-baseline --no-e2e > $O/tf32_$d.json 2> $O/tf32_$d.err; done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt

#!/bin/bash
mkdir -p gpurun_out/c7
O=gpurun_out/c7
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 900 python tools/exp_c5_l2.py > $O/exp_c5_l2.txt 2>&1
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err

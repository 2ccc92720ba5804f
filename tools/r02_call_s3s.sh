#!/bin/bash
mkdir -p gpurun_out/s3s
O=gpurun_out/s3s
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/c5.txt
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err

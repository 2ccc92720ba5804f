#!/bin/bash
mkdir -p gpurun_out/c11
O=gpurun_out/c11
timeout 600 python tools/exp_dropin.py > $O/exp_dropin.txt 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
HCS_PROFILE_TIMED=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -k c1_bench -p no:cacheprovider > $O/pytest_c1.txt 2>&1

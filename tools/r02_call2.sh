#!/bin/bash
# round 2 call 2: in-kernel split-unit completion (no fix-up launch): GPU tests, C1/C2 bench, C1 launch list
mkdir -p gpurun_out/c2
O=gpurun_out/c2
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --cuda-graph off > $O/bench_c1_nograph.json 2> $O/bench_c1_nograph.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c1.csv python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --cuda-graph off > /dev/null 2>&1
ls -la $O

#!/bin/bash
mkdir -p gpurun_out/c17
O=gpurun_out/c17
export HCS_PARITY_LOG=$PWD/$O/parity.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
unset HCS_PARITY_LOG
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 90 python tools/exp_c1.py > $O/exp_c1.txt 2>&1
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize.py > $O/racecheck.txt 2>&1; echo "rc=$?" >> $O/racecheck.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python tools/sanitize.py > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt

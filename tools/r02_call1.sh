#!/bin/bash
# round 2 (re-entry) call 1: validate the committed state on the B200: smoke, all GPU tests,
# default bench, reference arm, 2-rank shared-GPU bench, launch list of the default bench.
mkdir -p gpurun_out/c1
O=gpurun_out/c1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
export HCS_PARITY_LOG=$PWD/$O/parity.jsonl
timeout 1800 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.txt
unset HCS_PARITY_LOG
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/bench_ref.err
HCS_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_shared2.json 2> $O/bench_shared2.err; echo "shared2 rc=$?" >> $O/bench_shared2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la $O

#!/bin/bash
# round 2: full GPU tests after the racecheck fix + drop-in staging; default bench (C2 + e2e + dropin),
# reference arm (installed rowwin), C3 epoch bench + launch list, sanitizer racecheck re-run
mkdir -p gpurun_out/c10
O=gpurun_out/c10
export HCS_PARITY_LOG=$PWD/$O/parity.jsonl
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
unset HCS_PARITY_LOG
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "rc=$?" >> $O/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv -k regex:"." -s 400 -c 300 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 30 python tools/sanitize.py > $O/sanitizer_racecheck.txt 2>&1; echo "racecheck rc=$?" >> $O/sanitizer_racecheck.txt
ls -la $O

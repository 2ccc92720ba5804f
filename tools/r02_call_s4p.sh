#!/bin/bash
mkdir -p gpurun_out/s4p
O=gpurun_out/s4p
HCS_PROFILE_TIMED=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 > $O/ncu.log 2>&1
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/c3.json 2> $O/c3.err

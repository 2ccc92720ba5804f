#!/bin/bash
# final C3 epoch (CUDA graph replay): ncu launch list of one timed epoch
mkdir -p gpurun_out/s4o
O=gpurun_out/s4o
HCS_PROFILE_TIMED=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 > $O/ncu.log 2>&1

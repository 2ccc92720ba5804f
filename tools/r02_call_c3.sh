#!/bin/bash
# C3 explicit epoch: full GPU suite, ncu launch list of one timed epoch, sanitizer on the new kernels
mkdir -p gpurun_out/c3
O=gpurun_out/c3
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
HCS_PROFILE_TIMED=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 > /dev/null 2>&1
timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_gnn.py -x -q -m gpu -k "xent or bf16_operand" -p no:cacheprovider > $O/racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_gnn.py -x -q -m gpu -k "xent or bf16_operand" -p no:cacheprovider > $O/synccheck.txt 2>&1

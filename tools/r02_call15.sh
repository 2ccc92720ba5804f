#!/bin/bash
mkdir -p gpurun_out/c15
timeout 300 python tools/dbg_async.py > gpurun_out/c15/dbg.txt 2>&1
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_spmm.py -q -p no:cacheprovider > gpurun_out/c15/pytest_spmm_$i.txt 2>&1; done

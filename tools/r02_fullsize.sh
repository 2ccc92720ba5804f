#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=20 > gpurun_out/r02_fullsize.txt 2>&1
echo "rc=$?" >> gpurun_out/r02_fullsize.txt

#!/bin/bash
mkdir -p gpurun_out/c16
timeout 600 python -m pytest tests/test_gpu_spmm.py -q -p no:cacheprovider > gpurun_out/c16/pytest_spmm.txt 2>&1

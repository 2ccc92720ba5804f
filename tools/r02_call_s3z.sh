#!/bin/bash
mkdir -p gpurun_out/s3z
timeout 600 python -m pytest tests/test_gpu_spmm.py -q -x -p no:cacheprovider -k "entry_point" > gpurun_out/s3z/t.txt 2>&1; echo "rc=$?" >> gpurun_out/s3z/t.txt

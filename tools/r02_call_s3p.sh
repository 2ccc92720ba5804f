#!/bin/bash
mkdir -p gpurun_out/s3p
timeout 900 python -m pytest tests/test_gpu_spmm.py -q -x -p no:cacheprovider -k "balanced or grid" > gpurun_out/s3p/t.txt 2>&1; echo "rc=$?" >> gpurun_out/s3p/t.txt
timeout 600 python tools/sanitize.py > gpurun_out/s3p/san_plain.txt 2>&1; echo "rc=$?" >> gpurun_out/s3p/san_plain.txt

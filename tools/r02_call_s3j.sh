#!/bin/bash
mkdir -p gpurun_out/s3j
CFG=c5 timeout 900 python tools/exp_c5_shuffle.py > gpurun_out/s3j/shuf.txt 2>&1
CFG=c2 timeout 600 python tools/exp_c5_shuffle.py >> gpurun_out/s3j/shuf.txt 2>&1

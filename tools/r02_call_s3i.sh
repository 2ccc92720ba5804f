#!/bin/bash
mkdir -p gpurun_out/s3i
CFG=c2 timeout 600 python tools/exp_tile_balance.py > gpurun_out/s3i/bal.txt 2>&1
CFG=c5 timeout 600 python tools/exp_tile_balance.py >> gpurun_out/s3i/bal.txt 2>&1

#!/bin/bash
mkdir -p gpurun_out/s3k
CFG=c5 timeout 900 python tools/exp_tile_alpha.py > gpurun_out/s3k/alpha.txt 2>&1
CFG=c2 DIMS=64,128 timeout 600 python tools/exp_tile_alpha.py >> gpurun_out/s3k/alpha.txt 2>&1

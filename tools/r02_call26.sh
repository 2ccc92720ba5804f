#!/bin/bash
mkdir -p gpurun_out/c26
timeout 900 python tools/exp_c5_pf.py > gpurun_out/c26/exp_c5_pf.txt 2>&1
echo "== c2" >> gpurun_out/c26/exp_c5_pf.txt; DIMS=64,128 timeout 300 python tools/exp_tile_dims.py >> gpurun_out/c26/exp_c5_pf.txt 2>&1

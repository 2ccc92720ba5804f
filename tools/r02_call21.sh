#!/bin/bash
mkdir -p gpurun_out/c21
O=gpurun_out/c21
DIMS=128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_chunk -s 3 -c 1 -o $O/chunk python tools/exp_tile_dims.py > /dev/null 2>&1

#!/bin/bash
mkdir -p gpurun_out/c19
O=gpurun_out/c19
HCS_LIB_PATH=$PWD/tools/exp_libs/libhcspmm_nogather_nomma.so DIMS=128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_warp -s 3 -c 1 -o $O/nogather_nomma python tools/exp_tile_dims.py > /dev/null 2>&1
HCS_LIB_PATH=$PWD/tools/exp_libs/libhcspmm_nomma.so DIMS=128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_warp -s 3 -c 1 -o $O/nomma python tools/exp_tile_dims.py > /dev/null 2>&1
ls -la $O

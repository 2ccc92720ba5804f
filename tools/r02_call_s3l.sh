#!/bin/bash
mkdir -p gpurun_out/s3l
O=gpurun_out/s3l
H=tools/exp_libs/head/libhcspmm.so
echo "== head c2" >> $O/r.txt; HCS_LIB_PATH=$H DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/r.txt 2>&1
echo "== new c2 (alpha 64)" >> $O/r.txt; DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/r.txt 2>&1
echo "== head c2" >> $O/r.txt; HCS_LIB_PATH=$H DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/r.txt 2>&1
echo "== new c2 alpha sweep" >> $O/r.txt; CFG=c2 DIMS=128 ALPHAS=0,64,256,0,64 timeout 600 python tools/exp_tile_alpha.py 2>&1 | grep "^{" >> $O/r.txt
echo "== head c5" >> $O/r.txt; HCS_LIB_PATH=$H timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/r.txt
echo "== new c5 alpha sweep" >> $O/r.txt; CFG=c5 ALPHAS=0,64,256,1024,0,256 timeout 900 python tools/exp_tile_alpha.py 2>&1 | grep "^{" >> $O/r.txt

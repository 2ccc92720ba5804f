#!/bin/bash
mkdir -p gpurun_out/s3m
O=gpurun_out/s3m
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
echo "== head c2" >> $O/r.txt; HCS_LIB_PATH=tools/exp_libs/head/libhcspmm.so DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/r.txt 2>&1
echo "== new c2" >> $O/r.txt; DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/r.txt 2>&1
echo "== new c5" >> $O/r.txt; CFG=c5 ALPHAS=0,256,0,256 timeout 900 python tools/exp_tile_alpha.py 2>&1 | grep "^{" >> $O/r.txt
echo "== new c5 all" >> $O/r.txt; timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/r.txt

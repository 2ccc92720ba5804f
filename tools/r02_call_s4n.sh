#!/bin/bash
mkdir -p gpurun_out/s4n
CFG=c5 ALPHAS=256,128,192,384,512,256,384 timeout 1500 python tools/exp_tile_alpha.py 2>&1 | grep "^{" > gpurun_out/s4n/alpha.txt

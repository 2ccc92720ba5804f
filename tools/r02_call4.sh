#!/bin/bash
mkdir -p gpurun_out/c4
O=gpurun_out/c4
timeout 300 python tools/exp_c1.py > $O/exp_c1.txt 2>&1
DIM=32 timeout 300 python tools/exp_c1.py > $O/exp_c1_d32.txt 2>&1

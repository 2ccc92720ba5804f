#!/bin/bash
mkdir -p gpurun_out/s3g
O=gpurun_out/s3g
DIM=32 PREC=bf16 timeout 300 python tools/exp_c1.py > $O/c1.txt 2>&1
DIM=32 PREC=tf32 timeout 300 python tools/exp_c1.py >> $O/c1.txt 2>&1

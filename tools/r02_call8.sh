#!/bin/bash
mkdir -p gpurun_out/c8
O=gpurun_out/c8
timeout 900 python tools/exp_c5_l2.py > $O/exp_c5_l2.txt 2>&1

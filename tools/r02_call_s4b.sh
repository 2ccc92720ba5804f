#!/bin/bash
mkdir -p gpurun_out/s4b
O=gpurun_out/s4b
timeout 900 python -m pytest tests/test_gpu_spmm.py -q -x -p no:cacheprovider -k "ring or scalar" > $O/t.txt 2>&1; echo "rc=$?" >> $O/t.txt
echo "== auto (ring)" >> $O/c5.txt; timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/c5.txt
echo "== warp16" >> $O/c5.txt; C5_SCALAR_VARIANT=warp16 timeout 600 python tools/exp_c5.py 2>&1 | grep -v "^{" >> $O/c5.txt

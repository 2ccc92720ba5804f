#!/bin/bash
# Experiment (not product): warps per CTA of the 32-feature-slice tile kernel (N <= 32).
out=gpurun_out/tile_warps.log
: > $out
for w in 12 16 12 16; do
  touch paper_2412_08902_b200/csrc/spmm_tile_warp.cu
  HCS_NVCC_EXTRA="-DHCS_TILE_WARPS4=$w" python -m paper_2412_08902_b200._build > /tmp/b.log 2>&1 || { echo "build failed $w" >> $out; continue; }
  echo "warps4=$w $(DIMS=8,24,32 timeout 300 python tools/exp_tile_dims.py 2>&1 | tail -1)" >> $out
done
touch paper_2412_08902_b200/csrc/spmm_tile_warp.cu
python -m paper_2412_08902_b200._build > /dev/null 2>&1

#!/bin/bash
# ncu full capture of the warp-independent tile kernel (C2, dim 128 and 32)
mkdir -p gpurun_out
for d in 128 32; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_warp$ -s 2 -c 1 \
   -o gpurun_out/warp_d$d python bench.py --steps 3 --warmup 3 --dim $d --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
ls -la gpurun_out

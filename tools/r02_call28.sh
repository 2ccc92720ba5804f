#!/bin/bash
# round 2 evidence: ncu full captures of the C3 fused launches (paired epilogue) and of C5's tile and scalar launches
mkdir -p gpurun_out/c28
O=gpurun_out/c28
timeout 900 ncu --set full --clock-control none -k regex:k_tile_warp -s 6 -c 3 -o $O/fused_c3 python bench.py --config c3 --steps 1 --warmup 3 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"k_tile_warp|k_spmm_scalar_w" -s 4 -c 2 -o $O/c5 python tools/exp_c5.py > /dev/null 2>&1
ls -la $O

#!/bin/bash
mkdir -p gpurun_out/c25
O=gpurun_out/c25
echo "== warp2" > $O/dims.txt; DIMS=64,72,96,128 timeout 300 python tools/exp_tile_dims.py >> $O/dims.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_spmm.py -q -x -p no:cacheprovider -k "warp2 or pairing or graph_replay or async or slice_widths or tile_path_dims or feature_dims" > $O/pytest_w2.txt 2>&1

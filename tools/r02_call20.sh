#!/bin/bash
mkdir -p gpurun_out/c20
O=gpurun_out/c20
timeout 600 python -m pytest tests/test_gpu_spmm.py -q -x -p no:cacheprovider -k "chunk_kernel or pairing or graph_replay or async or slice_widths" > $O/pytest_chunk.txt 2>&1
echo "== chunk" > $O/dims.txt; DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/dims.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err

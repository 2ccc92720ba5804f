#!/bin/bash
mkdir -p gpurun_out/c32
timeout 600 python -m pytest tests/test_gpu_spmm.py -q -p no:cacheprovider -k "tile_grid or pairing" > gpurun_out/c32/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/c32/pytest.txt
HCS_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c32/bench_shared2.json 2> gpurun_out/c32/bench_shared2.err

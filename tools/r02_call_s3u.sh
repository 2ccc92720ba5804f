#!/bin/bash
mkdir -p gpurun_out/s3u
O=gpurun_out/s3u
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
DIM=32 PREC=bf16 timeout 300 python tools/exp_c1.py 2>&1 | cut -c1-200 > $O/c1.txt
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --precision tf32 --no-cpu-baseline > $O/bench_c1_tf32.json 2> $O/bench_c1_tf32.err
DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py > $O/c2.txt 2>&1

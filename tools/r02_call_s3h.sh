#!/bin/bash
mkdir -p gpurun_out/s3h
O=gpurun_out/s3h
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_ops.py tests/test_gpu_gnn.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
DIM=32 PREC=bf16 timeout 300 python tools/exp_c1.py > $O/c1.txt 2>&1
DIM=32 PREC=tf32 timeout 300 python tools/exp_c1.py >> $O/c1.txt 2>&1
timeout 600 python bench.py --config c1 --steps 200 --warmup 10 > $O/bench_c1.json 2> $O/bench_c1.err

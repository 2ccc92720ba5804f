#!/bin/bash
mkdir -p gpurun_out/c33
O=gpurun_out/c33
timeout 900 python -m pytest tests/test_gpu_gnn.py tests/test_gpu_ops.py tests/test_gpu_multirank.py -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err

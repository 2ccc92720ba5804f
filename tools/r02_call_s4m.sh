#!/bin/bash
mkdir -p gpurun_out/s4m
O=gpurun_out/s4m
timeout 900 python -m pytest tests/test_gpu_gnn.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider > $O/t.txt 2>&1; echo "rc=$?" >> $O/t.txt
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/c3.json 2> $O/c3.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/c3b.json 2> $O/c3b.err

#!/bin/bash
mkdir -p gpurun_out/s4h
O=gpurun_out/s4h
for rep in 1 2; do
echo "== new" >> $O/r.txt; timeout 300 python tools/exp_gemm.py >> $O/r.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_gnn.py -q -x -p no:cacheprovider > $O/t.txt 2>&1; echo "rc=$?" >> $O/t.txt
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/c3.json 2> $O/c3.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/c3b.json 2> $O/c3b.err

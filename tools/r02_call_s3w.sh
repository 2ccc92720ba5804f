#!/bin/bash
mkdir -p gpurun_out/s3w
O=gpurun_out/s3w
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/c3_graph.json 2> $O/c3_graph.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --cuda-graph off > $O/c3_eager.json 2> $O/c3_eager.err
timeout 1200 python -m pytest tests/test_gpu_gnn.py tests/test_gpu_multirank.py tests/test_gpu_ops.py -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt

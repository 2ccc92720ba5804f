#!/bin/bash
mkdir -p gpurun_out/s3v
O=gpurun_out/s3v
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/c3_graph.json 2> $O/c3_graph.err
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --cuda-graph off > $O/c3_eager.json 2> $O/c3_eager.err

#!/bin/bash
mkdir -p gpurun_out/s3x
timeout 600 python -m pytest tests/test_gpu_gnn.py -q -x -p no:cacheprovider -k "graph_replay" > gpurun_out/s3x/t.txt 2>&1; echo "rc=$?" >> gpurun_out/s3x/t.txt

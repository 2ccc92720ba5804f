#!/bin/bash
mkdir -p gpurun_out/s3c
O=gpurun_out/s3c
timeout 1200 python tools/exp_c5_hotorder.py > $O/hot.jsonl 2> $O/hot.err

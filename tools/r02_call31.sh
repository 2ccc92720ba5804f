#!/bin/bash
mkdir -p gpurun_out/c31
CFGS=c5,c2 timeout 2400 python tools/exp_shard_compute.py > gpurun_out/c31/shard_compute.txt 2>&1

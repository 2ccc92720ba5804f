#!/bin/bash
mkdir -p gpurun_out/s4j
timeout 2400 python tools/exp_shard_compute.py > gpurun_out/s4j/shard.txt 2> gpurun_out/s4j/shard.err

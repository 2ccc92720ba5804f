#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/exp_paths.py > gpurun_out/exp_paths.log 2>&1
cd tools/probe
for args in "ldg" "gather4 1" "gather4 4" "mma 0"; do echo "=== probe $args"; timeout 300 ./probe $args 2>&1 | tail -40; done > ../../gpurun_out/probe.log 2>&1
timeout 300 ./gather_smem > ../../gpurun_out/gather_smem.log 2>&1

#!/bin/bash
# round 2, call 1: gather4 scaling probe + GPU test suite (baseline state)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt
timeout 600 ./tools/probe/g4scale > gpurun_out/r02_g4scale.txt 2>&1
echo "g4scale rc=$?" >> gpurun_out/r02_g4scale.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu.txt 2>&1
echo "pytest rc=$?"

#!/bin/bash
cd tools/probe
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
for args in "mma 0" "mma 1" "mma 2" "gather4 1" "gather4 4" "ldg"; do
  echo "=== probe $args"
  timeout 300 ./probe $args 2>&1 | tail -60
done

#!/bin/bash
mkdir -p gpurun_out/s4i
O=gpurun_out/s4i
timeout 900 python bench.py --config c4 --graph community --steps 20 --warmup 3 > $O/c4c.json 2> $O/c4c.err
timeout 900 python bench.py --config c4 --steps 20 --warmup 3 > $O/c4.json 2> $O/c4.err
timeout 600 python bench.py --graph community --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $O/c2c.json 2> $O/c2c.err

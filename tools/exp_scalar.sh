#!/bin/bash
timeout 300 python tools/exp_paths.py > gpurun_out/exp_paths2.log 2>&1
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['ms_per_step'], d['roofline']['kernel_ms'])" >> gpurun_out/exp_paths2.log 2>&1
timeout 300 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_gnn.py -x -q 2>&1 | tail -2 >> gpurun_out/exp_paths2.log

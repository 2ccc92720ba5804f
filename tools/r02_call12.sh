#!/bin/bash
mkdir -p gpurun_out/c12
O=gpurun_out/c12
timeout 600 python tools/exp_dropin.py > $O/exp_dropin.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 300 python -m pytest tests/test_gpu_spmm.py -q -k "host_pipelined or async" -p no:cacheprovider > $O/pytest.txt 2>&1

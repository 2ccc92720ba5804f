#!/bin/bash
# Experiment (not product): C3 epoch and C2 N=40/48 with the NPR=3 kernel on (1) / off (0).
for v in 1 0 1 0; do
  r=$(timeout 300 python -c "
import runpy, sys
from paper_2412_08902_b200 import _lib
_lib.call('hcs_set_tile_npr3', $v)
sys.argv = ['bench.py', '--config', 'c3', '--steps', '20', '--warmup', '3']
runpy.run_path('bench.py', run_name='__main__')" 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  echo "npr3=$v c3_ms=$r"
done
NPR3=1 DIMS=40,41,48 timeout 300 python tools/exp_tile_dims.py
NPR3=0 DIMS=40,41,48 timeout 300 python tools/exp_tile_dims.py

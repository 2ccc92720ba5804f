#!/bin/bash
mkdir -p gpurun_out/c6
O=gpurun_out/c6
CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/dbg_rows.py > $O/dbg.txt 2>&1; echo "rc=$?" >> $O/dbg.txt
timeout 120 compute-sanitizer --tool memcheck python tools/dbg_rows.py > $O/dbg_memcheck.txt 2>&1; echo "rc=$?" >> $O/dbg_memcheck.txt

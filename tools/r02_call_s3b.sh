#!/bin/bash
# C5 hot-row compaction + persisting L2 window experiment, shipping lib and no-hint lib
mkdir -p gpurun_out/s3b
O=gpurun_out/s3b
timeout 900 python tools/exp_c5_persist.py > $O/ship.jsonl 2> $O/ship.err
HCS_LIB_PATH=tools/exp_libs/xpol_none/libhcspmm.so timeout 900 python tools/exp_c5_persist.py > $O/none.jsonl 2> $O/none.err

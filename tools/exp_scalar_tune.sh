#!/bin/bash
# Experiment (not product): K3 tuning constants on C5's scalar windows.  Rebuilds the library with
# -DHCS_SCALAR_U32=<entries in flight> -DHCS_SCALAR_MINB=<blocks per SM> and times tools/exp_c5.py.
out=gpurun_out/scalar_tune.log
: > $out
for cfg in "3 3" "4 3" "2 3" "3 4" "4 4" "2 4" "3 2" "6 2"; do
  set -- $cfg
  touch paper_2412_08902_b200/csrc/spmm_scalar.cu
  HCS_NVCC_EXTRA="-DHCS_SCALAR_U32=$1 -DHCS_SCALAR_MINB=$2" python -m paper_2412_08902_b200._build > /tmp/b.log 2>&1 || { echo "build failed $cfg" >> $out; cat /tmp/b.log >> $out; continue; }
  r=$(timeout 300 python tools/exp_c5.py 2>&1 | tail -1)
  echo "U=$1 MINB=$2 $r" >> $out
done
touch paper_2412_08902_b200/csrc/spmm_scalar.cu
python -m paper_2412_08902_b200._build > /dev/null 2>&1

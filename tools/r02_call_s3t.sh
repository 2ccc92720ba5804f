#!/bin/bash
mkdir -p gpurun_out/s3t
O=gpurun_out/s3t
for rep in 1 2; do
for v in default sg1 sg4; do
  if [ $v = default ]; then L=""; else L=tools/exp_libs/$v/libhcspmm.so; fi
  for p in bf16 tf32; do
  echo "== $v $p" >> $O/c1.txt; HCS_LIB_PATH=$L DIM=32 PREC=$p timeout 300 python tools/exp_c1.py 2>&1 | head -1 | cut -c1-150 >> $O/c1.txt
  done
done
done
for v in default sg1; do
  if [ $v = default ]; then L=""; else L=tools/exp_libs/$v/libhcspmm.so; fi
  HCS_LIB_PATH=$L timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $O/b_$v.json 2>/dev/null
  HCS_LIB_PATH=$L timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --precision tf32 > $O/bt_$v.json 2>/dev/null
done

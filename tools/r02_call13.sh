#!/bin/bash
mkdir -p gpurun_out/c13
O=gpurun_out/c13
for lib in default nosync w12 w12nosync; do
  if [ $lib = default ]; then unset HCS_LIB_PATH; else export HCS_LIB_PATH=$PWD/tools/exp_libs/libhcspmm_$lib.so; fi
  echo "== $lib" >> $O/dims.txt
  DIMS=32,64,128 timeout 300 python tools/exp_tile_dims.py >> $O/dims.txt 2>&1
done
unset HCS_LIB_PATH
timeout 900 python -m pytest tests/test_gpu_gnn.py tests/test_gpu_ops.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err

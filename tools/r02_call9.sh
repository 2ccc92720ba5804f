#!/bin/bash
# round 2: ncu full capture of the current tile kernel (C2 N=128), launch list of the default bench,
# compute-sanitizer passes over every product kernel (tools/sanitize.py)
mkdir -p gpurun_out/c9
O=gpurun_out/c9
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_warp -s 2 -c 1 -o $O/full_tile_c2_d128 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize.py > $O/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/sanitizer_$tool.txt
done
ls -la $O

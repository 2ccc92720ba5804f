#!/bin/bash
# round 2 call b: GPU tests after the K7/tf32-fused/dense changes, reference arm, sanitizers
mkdir -p gpurun_out
export HCS_PARITY_LOG=$PWD/gpurun_out/r02_parity.jsonl
rm -f $HCS_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
echo "ref rc=$?" >> gpurun_out/r02_bench_ref.err
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/r02_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02_sanitizer_$tool.txt
done

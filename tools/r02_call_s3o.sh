#!/bin/bash
mkdir -p gpurun_out/s3o
O=gpurun_out/s3o
for t in memcheck racecheck synccheck; do
  echo "== $t" >> $O/san.txt
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize.py >> $O/san.txt 2>&1; echo "$t rc=$?" >> $O/san.txt
done

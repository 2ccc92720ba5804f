#!/bin/bash
mkdir -p gpurun_out
G4_WIDE=1 timeout 600 ./tools/probe/g4scale > gpurun_out/r02_g4scale_wide.txt 2>&1
echo "rc=$?" >> gpurun_out/r02_g4scale_wide.txt

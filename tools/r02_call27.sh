#!/bin/bash
mkdir -p gpurun_out/c27
timeout 600 python -m pytest tests/test_gpu_spmm.py -q -p no:cacheprovider -k "pieces_wide or scalar_variants or degenerate" > gpurun_out/c27/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/c27/pytest.txt

#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_full_parity.py -q -x > gpurun_out/t17.log 2>&1; tail -15 gpurun_out/t17.log
timeout 1500 python scripts/variant_timing.py libhcb.so,libhcb_nolive.so er25,rmat22,rmat26,rmat17 > gpurun_out/t17.txt 2>&1
cat gpurun_out/t17.txt

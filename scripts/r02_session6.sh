#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > gpurun_out/t6.log 2>&1; tail -3 gpurun_out/t6.log
timeout 900 python scripts/variant_timing.py libhcb.so,libhcb.so:ell=0 grid4096,grid2048 > gpurun_out/t6_timing.txt 2>&1
cat gpurun_out/t6_timing.txt

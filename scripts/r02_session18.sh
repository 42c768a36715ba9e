#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 300 python scripts/live_debug.py > gpurun_out/t22.log 2>&1
for K in dense_core hubs mixed_degrees rmat; do timeout 300 python scripts/fuzz_debug.py $K 16 2>&1 | tail -3; done >> gpurun_out/t22.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_full_parity.py -q -x >> gpurun_out/t22.log 2>&1; tail -25 gpurun_out/t22.log
timeout 1500 python scripts/variant_timing.py libhcb.so,libhcb_nostage.so er25,rmat22,rmat26,rmat16 > gpurun_out/t22.txt 2>&1
cat gpurun_out/t22.txt

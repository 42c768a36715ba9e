#!/usr/bin/env bash
set -u
timeout 300 python scripts/live_debug.py > gpurun_out/t33.log 2>&1; grep -c " ok " gpurun_out/t33.log; grep -v " ok " gpurun_out/t33.log | head
for K in hubs dense_core rmat mixed_degrees; do timeout 300 python scripts/fuzz_debug.py $K 12 2>&1 | tail -2; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_full_parity.py -q -x 2>&1 | tail -2
timeout 900 python scripts/variant_timing.py libhcb.so,libhcb_nodefer.so rmat22,rmat26,rmat16,er25 > gpurun_out/t33.txt 2>&1; cat gpurun_out/t33.txt

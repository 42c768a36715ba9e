#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_full_parity.py tests/test_mg_peer.py -q -x > gpurun_out/t14.log 2>&1; tail -3 gpurun_out/t14.log
timeout 1500 python scripts/variant_timing.py libhcb.so,libhcb_k0.so,libhcb_k25.so,libhcb_k100.so rmat16,rmat22,rmat26,er25 > gpurun_out/t14.txt 2>&1
cat gpurun_out/t14.txt

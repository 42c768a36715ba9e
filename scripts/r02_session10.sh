#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_full_parity.py tests/test_mg_peer.py -q -x > gpurun_out/t11.log 2>&1; tail -3 gpurun_out/t11.log
timeout 900 python scripts/variant_timing.py libhcb.so er25,grid4096,rmat22,rmat16,rmat26 > gpurun_out/t11_timing.txt 2>&1
cat gpurun_out/t11_timing.txt
HCB_LIB=libhcb_pt.so timeout 300 python scripts/phase_times.py rmat22 > gpurun_out/t11_pt.txt 2>&1; head -30 gpurun_out/t11_pt.txt

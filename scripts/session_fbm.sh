#!/usr/bin/env bash
# GPU session: parity of the bitmap-assign solver, then A/B timing against the
# round-1 solver (libhcb_orig.so).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fbm_smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/fbm_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fbm_tests.log
tail -15 gpurun_out/fbm_tests.log
timeout 1500 python scripts/variant_timing.py libhcb_orig.so,libhcb.so grid4096,er25,rmat22,rmat16,rmat26 > gpurun_out/fbm_ab.txt 2>&1
cat gpurun_out/fbm_ab.txt

#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 1500 python scripts/variant_timing.py libhcb.so,libhcb_wc.so,libhcb_fb.so,libhcb_wcfb.so grid4096,rmat16,rmat22,er25 > gpurun_out/t12.txt 2>&1
cat gpurun_out/t12.txt

#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 1500 python scripts/variant_timing.py libhcb.so,libhcb_filt.so,libhcb_hint.so,libhcb_fh.so er25,grid4096,rmat22,rmat16,rmat26 > gpurun_out/ab_push.txt 2>&1
cat gpurun_out/ab_push.txt

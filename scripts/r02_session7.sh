#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 900 python scripts/variant_timing.py libhcb.so,libhcb.so:l2=0,libhcb_n4p1.so,libhcb_n4p2.so,libhcb_m4.so grid4096 > gpurun_out/t7_timing.txt 2>&1
cat gpurun_out/t7_timing.txt

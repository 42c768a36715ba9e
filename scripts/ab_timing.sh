#!/usr/bin/env bash
# A/B solve timing of in-tree builds: scripts/ab_timing.sh "libhcb_orig.so,libhcb.so" grid4096,er25,rmat22,rmat16
# (min of 3 L2-flushed solves per mode; writes gpurun_out/<tag>.txt)
set -u
LIBS=${1:-libhcb.so}
CFGS=${2:-grid4096,er25,rmat22,rmat16}
TAG=${3:-ab}
mkdir -p gpurun_out
timeout 1500 python scripts/variant_timing.py "$LIBS" "$CFGS" 2>&1 | tee gpurun_out/${TAG}.txt

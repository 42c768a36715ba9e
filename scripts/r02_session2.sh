#!/usr/bin/env bash
# Round-2 GPU session 2: GPU suite after the odd-m fix, bitmap vs scan assign A/B, ncu of ER-2^25.
set -u
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -q -m gpu -x ) > gpurun_out/gpu_tests2.log 2>&1
tail -8 gpurun_out/gpu_tests2.log
timeout 1200 python scripts/variant_timing.py libhcb.so,libhcb_scan.so er25,grid4096,rmat22,rmat16 > gpurun_out/ab_fbm.txt 2>&1
cat gpurun_out/ab_fbm.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve_kernel -s 1 -c 1 \
   -o gpurun_out/er25_fbm_full python scripts/ncu_solve.py er25 hybrid 2 > gpurun_out/ncu_er25.log 2>&1
tail -3 gpurun_out/ncu_er25.log
HCB_LIB=libhcb_scan.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve_kernel -s 1 -c 1 \
   -o gpurun_out/er25_scan_full python scripts/ncu_solve.py er25 hybrid 2 > gpurun_out/ncu_er25s.log 2>&1
tail -3 gpurun_out/ncu_er25s.log

#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_full_parity.py -q -x > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
timeout 1200 python scripts/variant_timing.py libhcb.so,libhcb_nopersist.so er25,grid4096,rmat22,rmat16,rmat26 > gpurun_out/ab_persist.txt 2>&1
cat gpurun_out/ab_persist.txt
timeout 600 python scripts/rounds.py rmat16 er25 rmat22 grid4096 > gpurun_out/rounds4.txt 2>&1
for c in er25 grid4096 rmat16; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve_kernel -s 1 -c 1 \
   -o gpurun_out/${c}_r02_full python scripts/ncu_solve.py $c hybrid 2 > gpurun_out/ncu_$c.log 2>&1
tail -1 gpurun_out/ncu_$c.log
done

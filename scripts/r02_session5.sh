#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_full_parity.py -q -x > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
timeout 900 python scripts/variant_timing.py libhcb.so er25,grid4096,rmat22,rmat16,rmat26 > gpurun_out/t5_timing.txt 2>&1
cat gpurun_out/t5_timing.txt
timeout 600 python scripts/rounds.py rmat16 er25 rmat22 grid4096 > gpurun_out/rounds5.txt 2>&1
for c in er25 grid4096 rmat16 rmat22; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve_kernel -s 1 -c 1 \
   -o /tmp/${c}_r02 python scripts/ncu_solve.py $c hybrid 2 > gpurun_out/ncu_$c.log 2>&1
python scripts/ncu_summary.py /tmp/${c}_r02.ncu-rep > gpurun_out/ncu_${c}_summary.txt 2>&1
python scripts/ncu_lines.py /tmp/${c}_r02.ncu-rep 40 > gpurun_out/ncu_${c}_lines.txt 2>&1
done
cp /tmp/grid4096_r02.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out

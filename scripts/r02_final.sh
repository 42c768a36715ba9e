#!/usr/bin/env bash
# Round-2 closing measurement session on one B200 (outputs under gpurun_out/r02c/):
# GPU suite + smoke, DRAM traffic of one solve_kernel launch per config
# (copied into profiles/ first so the bench line carries it), the bench line
# (every config), the reference arm, the launch list of the headline step,
# ncu --set full summaries of three configs.
set -u
O=gpurun_out/r02c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 200 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1
for CFG in grid4096 rmat16 rmat22 er25 rmat26; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:solve_kernel -s 3 -c 1 --csv --log-file $O/r02_${CFG}_traffic.csv \
    python scripts/ncu_solve.py $CFG hybrid 4 > /dev/null 2>&1
  cp $O/r02_${CFG}_traffic.csv profiles/
done
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/reference_grid4096.json 2> $O/reference_grid4096.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_grid4096.csv \
  python bench.py --steps 2 --warmup 3 --skip-modes --skip-cpu --headline-only > /dev/null 2>&1
python scripts/launch_summary.py $O/launches_grid4096.csv > $O/launches_grid4096.txt 2>&1
for CFG in grid4096 er25 rmat26; do
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:solve_kernel -s 1 -c 1 -o /tmp/${CFG}_full \
    python scripts/ncu_solve.py $CFG hybrid 2 > /dev/null 2>&1
  python scripts/ncu_summary.py /tmp/${CFG}_full.ncu-rep > $O/ncu_full_${CFG}.txt 2>&1
  python scripts/ncu_lines.py /tmp/${CFG}_full.ncu-rep 30 >> $O/ncu_full_${CFG}.txt 2>&1
done
true
ls -la $O

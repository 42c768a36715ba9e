#!/usr/bin/env bash
# Refresh after a bin-0-only-kernel change: GPU suite + smoke, the grid's
# traffic capture (copied into profiles/ before the bench reads it), the bench
# line (every config), the grid launch list and ncu --set full (gpurun_out/r02e/).
set -u
O=gpurun_out/r02e
mkdir -p $O
timeout 200 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $O/gpu_tests.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:solve_kernel -s 3 -c 1 --csv --log-file $O/r02_grid4096_traffic.csv \
  python scripts/ncu_solve.py grid4096 hybrid 4 > /dev/null 2>&1
cp $O/r02_grid4096_traffic.csv profiles/
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_grid4096.csv \
  python bench.py --steps 2 --warmup 3 --skip-modes --skip-cpu --headline-only > /dev/null 2>&1
python scripts/launch_summary.py $O/launches_grid4096.csv > $O/launches_grid4096.txt 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:solve_kernel -s 1 -c 1 -o /tmp/grid4096_full \
  python scripts/ncu_solve.py grid4096 hybrid 2 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/grid4096_full.ncu-rep > $O/ncu_full_grid4096.txt 2>&1
python scripts/ncu_lines.py /tmp/grid4096_full.ncu-rep 30 >> $O/ncu_full_grid4096.txt 2>&1
ls -la $O

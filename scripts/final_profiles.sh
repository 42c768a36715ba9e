#!/usr/bin/env bash
# Round-end measurement session on one B200: every BASELINE config through
# bench.py, the reference arm, the launch list + DRAM traffic + a full ncu
# capture of the headline solve kernel.  Outputs under gpurun_out/final/.
set -u
O=gpurun_out/final
mkdir -p $O
timeout 200 python __graft_entry__.py smoke > $O/smoke.txt 2>&1
for CFG in grid4096 rmat16 rmat22 er25 rmat26; do
  timeout 1200 python bench.py --config $CFG --steps 5 --warmup 3 > $O/bench_$CFG.json 2> $O/bench_$CFG.err
done
timeout 600 python bench.py --impl reference --config grid4096 --steps 3 --warmup 3 > $O/reference_grid4096.json 2> $O/reference_grid4096.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_grid4096.csv \
  python bench.py --config grid4096 --steps 2 --warmup 3 --skip-modes --skip-cpu > /dev/null 2>&1
for CFG in grid4096 rmat22 er25; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:solve_kernel -s 3 -c 1 --csv --log-file $O/traffic_$CFG.csv \
    python scripts/ncu_solve.py $CFG hybrid 4 > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve_kernel -s 1 -c 1 -o $O/grid_full \
  python scripts/ncu_solve.py grid4096 hybrid 2 > /dev/null 2>&1
ls -la $O

#!/usr/bin/env bash
# One GPU-box session: tests, smoke, bench (JSON), launch list + DRAM traffic
# of the solve kernel (ncu), copied under gpurun_out/.  Dev helper.
CFG=${1:-grid4096}
timeout 200 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py --config $CFG --steps 5 --warmup 3 > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err
tail -c 2500 gpurun_out/bench_$CFG.json; tail -3 gpurun_out/bench_$CFG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 2 --warmup 3 --skip-modes --skip-cpu > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:solve_kernel -s 3 -c 1 --csv --log-file gpurun_out/traffic_$CFG.csv python scripts/ncu_solve.py $CFG hybrid 4 > /dev/null 2>&1
tail -5 gpurun_out/traffic_$CFG.csv

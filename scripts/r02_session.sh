#!/usr/bin/env bash
# Round-2 GPU session: smoke, GPU suite, default bench (all configs), reference arm.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/smi.txt 2>&1
nproc >> gpurun_out/smi.txt; lscpu | grep "Model name" >> gpurun_out/smi.txt
( time timeout 300 python __graft_entry__.py smoke ) > gpurun_out/smoke.log 2>&1
tail -3 gpurun_out/smoke.log
( time timeout 2400 python -m pytest tests -q -m gpu --durations=25 ) > gpurun_out/gpu_tests.log 2>&1
tail -40 gpurun_out/gpu_tests.log
( time timeout 1500 python bench.py ) > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err

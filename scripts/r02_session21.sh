#!/usr/bin/env bash
set -u
mkdir -p gpurun_out/sanitize2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "planned or forced" > gpurun_out/t21.log 2>&1; tail -15 gpurun_out/t21.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitize2/racecheck.log 2>&1
tail -3 gpurun_out/sanitize2/racecheck.log

#!/usr/bin/env bash
# Quick A/B of the current build (dev aid): GPU parity subset, then the
# hybrid ms/step of each config given (default: all five), no modes, no CPU leg.
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_full_parity.py > gpurun_out/ab_tests.log 2>&1; tail -2 gpurun_out/ab_tests.log
for c in ${@:-rmat16 grid4096 rmat22 er25 rmat26}; do
  timeout 600 python bench.py --config $c --headline-only --skip-cpu --skip-modes > gpurun_out/ab_$c.json 2> gpurun_out/ab_$c.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step'],3), [round(x,3) for x in d.get('step_ms',[])])" || tail -3 gpurun_out/ab_$c.err
done

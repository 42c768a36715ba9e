#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_run.py
set -u
O=gpurun_out/sanitize
mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/summary.txt
  tail -3 $O/$tool.log >> $O/summary.txt
done
cat $O/summary.txt

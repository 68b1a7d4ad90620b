#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_run.py (one GPU): memcheck, racecheck, synccheck
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done

#!/usr/bin/env bash
# configs[4] batch throughput A/B: batch_ab.sh TAG "ENV1" "ENV2" ...  (env assignments)
TAG=$1; shift
mkdir -p gpurun_out
for r in 1 2; do
for E in "$@"; do
  echo "== [$E]" >> gpurun_out/batch_ab_$TAG.txt
  env $E timeout 600 python tools/batch_host.py 2>&1 | head -1 >> gpurun_out/batch_ab_$TAG.txt
done; done

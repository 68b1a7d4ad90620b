#!/usr/bin/env bash
# same-box A/B of the planner's CC path on the headline (6-primitive table):
# broad phase (auto, -1) vs the lockstep order (0)
mkdir -p gpurun_out; rm -f gpurun_out/bp_ab.log
for r in 1 2 3; do
  for bp in -1 0; do
    timeout 300 python bench.py --steps 4 --warmup 2 --no-extras --no-cpu --cc-broadphase $bp > gpurun_out/ab_tmp.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_tmp.json')); print('bp $bp', round(d['value'],4), round(d['p10_ms'],4), round(d['p90_ms'],4), round(d['e2e']['value'],4))" >> gpurun_out/bp_ab.log
  done
done

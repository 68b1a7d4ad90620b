#!/usr/bin/env bash
# same-box single-query team-count A/B on the headline workload: tools/team_ab.sh "160 192 224" [rounds]
T="${1:-160 192 224}"; R=${2:-2}
mkdir -p gpurun_out; rm -f gpurun_out/team_ab.log
for r in $(seq $R); do
  for t in $T; do
    timeout 300 python bench.py --steps 4 --warmup 2 --no-extras --no-cpu --teams $t > gpurun_out/ab_tmp.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_tmp.json')); print('teams $t', round(d['value'],4), round(d['p10_ms'],4), round(d['p90_ms'],4), round(d['e2e']['value'],4))" >> gpurun_out/team_ab.log
  done
done

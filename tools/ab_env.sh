#!/usr/bin/env bash
# same-box A/B of host/device knobs given as environment assignments:
#   tools/ab_env.sh "VAR=1 VAR2=x" "VAR=0" [rounds]   -> gpurun_out/ab.log
# (prints median / p10 / p90 / e2e per run; "" = the default build)
A="$1"; B="$2"; R=${3:-2}
for r in $(seq $R); do
  for v in A B; do
    if [ $v = A ]; then E="$A"; else E="$B"; fi
    env $E timeout 300 python bench.py --steps 4 --warmup 2 --no-extras --no-cpu > gpurun_out/ab_tmp.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_tmp.json')); print('$v [$E]', round(d['value'],4), round(d['p10_ms'],4), round(d['p90_ms'],4), round(d['e2e']['value'],4))" >> gpurun_out/ab.log
  done
done

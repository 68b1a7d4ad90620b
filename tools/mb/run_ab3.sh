#!/usr/bin/env bash
# stage-1 microbenchmark + planner A/B + projection parity for stage-1 variants
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
TAG=$1; shift
i=0
for D in "$@"; do
  i=$((i+1))
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -ftz=true -prec-div=false -prec-sqrt=false $(echo "$D" | sed 's/\([A-Z_0-9]*=[0-9]*\)/-D\1/g; s/,/ /g') \
       -DTU='"../../cprrtc-plan-g16-k0-o1.cu"' -o /tmp/stage1_bench_$i tools/mb/stage1_bench.cu 2>&1 | grep -i " error"
  echo "== [$D]" >> gpurun_out/mb_$TAG.txt
  /tmp/stage1_bench_$i | grep -E "stage1|damped|stop word none" >> gpurun_out/mb_$TAG.txt 2>&1
  CPRRTC_DEFINES="$D" timeout 600 python -m pytest tests/test_gpu_parity.py::test_projection_contract tests/test_gpu_steps.py -q -s -p no:cacheprovider 2>&1 | grep -E "agreement|passed|failed" >> gpurun_out/mb_$TAG.txt
done
for r in 1 2; do
  for D in "$@"; do
    CPRRTC_DEFINES="$D" timeout 300 python bench.py --steps 4 --warmup 2 --no-extras --no-cpu > gpurun_out/ab_tmp.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_tmp.json')); print('[$D]', round(d['value'],4), round(d['p10_ms'],4), round(d['p90_ms'],4), round(d['e2e']['value'],4))" >> gpurun_out/mb_$TAG.txt
  done
done

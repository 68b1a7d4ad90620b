#!/usr/bin/env bash
# stage-1 microbenchmark for two -D variants: run_ab.sh TAG "DEFS_A" "DEFS_B"
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for v in A B; do
  if [ $v = A ]; then D="$2"; else D="$3"; fi
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -ftz=true -prec-div=false -prec-sqrt=false $D \
       -DTU='"../../cprrtc-plan-g16-k0-o1.cu"' -o /tmp/stage1_bench_$v tools/mb/stage1_bench.cu 2>&1 | grep -i " error"
  echo "== $v [$D]" >> gpurun_out/mb_$1.txt
  /tmp/stage1_bench_$v >> gpurun_out/mb_$1.txt 2>&1
done

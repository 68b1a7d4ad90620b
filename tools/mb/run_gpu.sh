#!/usr/bin/env bash
# build (on the box, against the shipped TU) and run the stage-1 microbenchmark
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -ftz=true -prec-div=false -prec-sqrt=false \
     -DTU='"../../cprrtc-plan-g16-k0-o1.cu"' -o /tmp/stage1_bench tools/mb/stage1_bench.cu 2>&1 | grep -i " error"
/tmp/stage1_bench > gpurun_out/mb_${1:-x}.txt 2>&1

#!/usr/bin/env bash
# build the stage-1 microbenchmark against the current device source (no GPU needed to build)
set -e
cd "$(dirname "$0")/../.."
make -s -C paper_2505_06791_b200/csrc PY=python
python tools/dump_src.py > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -DTU='"../../cprrtc-plan-g16-k0-o1.cu"' \
     --use_fast_math -o stage1_bench tools/mb/stage1_bench.cu 2>&1 | grep -i " error" || true

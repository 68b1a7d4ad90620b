#!/usr/bin/env bash
# tests + bench (+ optional ncu of one kernel regex $2) on one B200; TAG = $1
TAG=${1:-q}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rA > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_$TAG.log
timeout 1500 python bench.py --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
if [ -n "$2" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 1 -c 1 \
    -o gpurun_out/prof_k_$TAG python bench.py --steps 1 --warmup 0 --queries 1 --no-cpu > gpurun_out/ncu_k_$TAG.log 2>&1
fi

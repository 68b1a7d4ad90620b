#!/usr/bin/env bash
TAG=${1:-s}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rA > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_$TAG.log
timeout 1500 python bench.py --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python tools/batch_host.py > gpurun_out/batch_host_$TAG.txt 2>&1
bash tools/sanitize.sh

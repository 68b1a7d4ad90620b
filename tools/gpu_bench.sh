#!/usr/bin/env bash
# default bench + reference arm on one B200 (outputs under gpurun_out/)
mkdir -p gpurun_out
TAG=${1:-x}
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
cp -r bench_records gpurun_out/bench_records_$TAG 2>/dev/null
timeout 900 python bench.py --impl reference > gpurun_out/reference_$TAG.json 2> gpurun_out/reference_$TAG.err

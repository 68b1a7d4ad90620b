#!/usr/bin/env bash
# ncu captures for profiles/ (run under gpurun; one GPU).
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --queries 5 --no-extras --no-cpu > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_plan_kernel -s 3 -c 1 \
    -o gpurun_out/prof_plan python bench.py --steps 1 --warmup 0 --queries 4 --no-extras --no-cpu > gpurun_out/ncu_plan.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_validate_kernel -s 1 -c 1 \
    -o gpurun_out/prof_cc python bench.py --steps 1 --warmup 0 --queries 1 --no-cpu > gpurun_out/ncu_cc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_nearest_kernel -s 1 -c 1 \
    -o gpurun_out/prof_nn python bench.py --steps 1 --warmup 0 --queries 1 --no-cpu > gpurun_out/ncu_nn.log 2>&1
ls -la gpurun_out

#!/usr/bin/env bash
# ncu captures for profiles/ (run under gpurun; one GPU).  Usage: tools/profile.sh <tag>
TAG=${1:-r1}
mkdir -p gpurun_out
python tools/dump_src.py > /dev/null && cp cprrtc-*.cu gpurun_out/
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 1 --queries 5 --no-extras --no-cpu > gpurun_out/ncu_launches_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_plan_kernel -s 3 -c 1 \
    -o gpurun_out/prof_plan_$TAG python tools/profile_plan.py > gpurun_out/ncu_plan_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'cp_validate_kernel' -s 1 -c 1 \
    -o gpurun_out/prof_cc_$TAG python bench.py --steps 1 --warmup 0 --queries 1 --no-cpu > gpurun_out/ncu_cc_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_validate_cull_kernel -s 1 -c 1 \
    -o gpurun_out/prof_cull_$TAG python bench.py --steps 1 --warmup 0 --queries 1 --no-cpu > gpurun_out/ncu_cull_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_nearest_kernel -s 1 -c 1 \
    -o gpurun_out/prof_nn_$TAG python bench.py --steps 1 --warmup 0 --queries 1 --no-cpu > gpurun_out/ncu_nn_$TAG.log 2>&1

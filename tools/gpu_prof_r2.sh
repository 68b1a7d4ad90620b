#!/usr/bin/env bash
# r2 profiling session: append-order A/B, ncu full capture of the plan kernel with source, launch list
mkdir -p gpurun_out
TAG=${1:-r2d}
rm -f gpurun_out/ab.log
bash tools/ab.sh "CP_APPEND_ORDER=0" "" 3
bash tools/ab.sh "CP_APPEND_ORDER=1" "" 2
python tools/dump_src.py > /dev/null && cp cprrtc-*.cu gpurun_out/
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_plan_kernel -s 3 -c 1 \
    -o gpurun_out/prof_plan_$TAG python tools/profile_plan.py > gpurun_out/ncu_plan_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 1 --queries 5 --no-extras --no-cpu > gpurun_out/ncu_launches_$TAG.log 2>&1

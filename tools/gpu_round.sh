#!/usr/bin/env bash
# tests + profile of the plan kernel at the default (512 teams) and full occupancy
timeout 1000 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_plan.py > gpurun_out/profile_plan_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cp_plan_kernel -s 3 -c 1 \
    -o gpurun_out/prof_plan512 python tools/profile_plan.py > gpurun_out/ncu_plan512.log 2>&1
TEAMS=2368 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cp_plan_kernel -s 3 -c 1 \
    -o gpurun_out/prof_planfull python tools/profile_plan.py > gpurun_out/ncu_planfull.log 2>&1

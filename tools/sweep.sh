#!/usr/bin/env bash
for t in 256 512 1024 0; do
  timeout 300 python bench.py --steps 2 --warmup 1 --queries 25 --no-extras --no-cpu --teams $t > gpurun_out/sweep_$t.json 2> gpurun_out/sweep_$t.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cp_plan_kernel -s 3 -c 1 \
    -o gpurun_out/prof_plan2 python bench.py --steps 1 --warmup 0 --queries 4 --no-extras --no-cpu > gpurun_out/ncu_plan2.log 2>&1

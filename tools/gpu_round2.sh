#!/usr/bin/env bash
# tests + bench + reference arm + ncu (plan, validate, cull, nn) on one B200; TAG = $1
TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rA > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
cp -r bench_records gpurun_out/bench_records_$TAG 2>/dev/null
timeout 900 python bench.py --impl reference > gpurun_out/reference_$TAG.json 2> gpurun_out/reference_$TAG.err
python tools/dump_src.py > /dev/null && cp cprrtc-*.cu gpurun_out/
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

#!/usr/bin/env bash
# same-box A/B: single-query P warps wait for the init grid after their first projection (CP_DEFER_WAIT)
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
bash tools/ab.sh "" "CP_DEFER_WAIT=1" 4
CPRRTC_DEFINES="CP_DEFER_WAIT=1" timeout 900 python -m pytest tests/test_gpu_planner.py tests/test_gpu_dropin.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_defer.log 2>&1; echo rc=$? >> gpurun_out/pytest_defer.log
CPRRTC_DEFINES="CP_DEFER_WAIT=1" timeout 600 python tools/soak.py 3 1 2 > gpurun_out/soak_defer.txt 2>&1; echo rc=$? >> gpurun_out/soak_defer.txt

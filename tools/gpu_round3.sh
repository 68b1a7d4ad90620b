#!/usr/bin/env bash
# full GPU round on one B200: tests, smoke, bench, reference arm, launch list, ncu of the
# plan / CC / NN kernels, soak, teardown timeline, sanitizers; TAG = $1
TAG=${1:-r2w}
bash tools/gpu_round2.sh $TAG
timeout 900 python tools/soak.py > gpurun_out/soak_$TAG.txt 2>&1; echo rc=$? >> gpurun_out/soak_$TAG.txt
timeout 600 python tools/teardown.py > gpurun_out/teardown_$TAG.txt 2>&1; echo rc=$? >> gpurun_out/teardown_$TAG.txt
bash tools/sanitize.sh
for t in memcheck racecheck synccheck; do cp gpurun_out/sanitize_$t.log gpurun_out/sanitize_${t}_$TAG.log; done

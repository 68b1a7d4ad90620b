#!/usr/bin/env bash
# CC kernel (999-box shelf, lockstep, flag off) checks/s for CPRRTC_DEFINES variants: cc_ab.sh TAG "D1" "D2" ...
TAG=$1; shift
mkdir -p gpurun_out
for r in 1 2; do
for D in "$@"; do
CPRRTC_DEFINES="$D" python - >> gpurun_out/cc_ab_$TAG.txt 2>&1 <<PY
import sys; sys.path[:0]=['.','tests']
import numpy as np, fixtures as fx, bench
from paper_2505_06791_b200 import kernels
m=fx.robot('arm7'); sc=fx.scene('shelf_x111')
wps=bench.cc_motions(m,16384,16)
kernels.validate_batch(m, sc, wps[:64], False)
best=min((kernels.validate_batch(m, sc, wps, False) for _ in range(5)), key=lambda r: r['kernel_ms'])
print('[$D]', round(best['gpu_checks'].sum()/(best['kernel_ms']*1e-3)/1e12, 4), 'T checks/s', round(best['kernel_ms'],4), 'ms')
PY
done; done

#!/usr/bin/env bash
# broad-phase CC (999-box shelf, flag on) reference checks resolved/s for CPRRTC_DEFINES variants
TAG=$1; shift
mkdir -p gpurun_out
for r in 1 2; do
for D in "$@"; do
CPRRTC_DEFINES="$D" python - >> gpurun_out/cull_ab_$TAG.txt 2>&1 <<PY
import sys; sys.path[:0]=['.','tests']
import numpy as np, fixtures as fx, bench
from paper_2505_06791_b200 import kernels
m=fx.robot('arm7')
for scn in ('shelf_x111', 'table'):
    sc=fx.scene(scn)
    wps=bench.cc_motions(m,16384,16)
    kernels.validate_batch(m, sc, wps[:64], True, broadphase=True)
    on=kernels.validate_batch(m, sc, wps, True)
    best=min((kernels.validate_batch(m, sc, wps, True, broadphase=True) for _ in range(5)), key=lambda r: r['kernel_ms'])
    assert (best['valid']==on['valid']).mean() > 0.99
    print('[$D]', scn, round(on['possible'].sum()/(best['kernel_ms']*1e-3)/1e12, 3), 'T resolved/s', round(best['kernel_ms'],4), 'ms')
PY
done; done

#!/usr/bin/env bash
# same-box A/B: round 0's connect from tree b's root (CP_ROOT_FIRST_CONNECT) vs the NN scan
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
bash tools/ab.sh "" "CP_ROOT_FIRST_CONNECT=1" 4

#!/usr/bin/env bash
# same-box A/B: round 0's extension from tree a's root (CP_ROOT_FIRST, default) vs the NN scan
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
bash tools/ab.sh "" "CP_ROOT_FIRST=0" 3

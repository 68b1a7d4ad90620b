#!/usr/bin/env bash
# GPU test suite (and optional extra args) on one B200; log under gpurun_out/
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rA "$@" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log

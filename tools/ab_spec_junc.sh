mkdir -p gpurun_out; rm -f gpurun_out/ab.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_spec.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_spec.log
bash tools/ab.sh "CP_SPEC_JUNC=0" "" 3
timeout 600 python tools/soak.py 300 2 > gpurun_out/soak_spec.txt 2>&1; echo rc=$? >> gpurun_out/soak_spec.txt

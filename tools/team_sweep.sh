mkdir -p gpurun_out; rm -f gpurun_out/sweep.log
for r in 1 2; do
for T in ${TEAMS:-256 296 370 444 222}; do
  timeout 300 python bench.py --steps 4 --warmup 2 --no-extras --no-cpu --teams $T > gpurun_out/sw_tmp.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw_tmp.json')); print('teams $T', round(d['value'],4), round(d['p10_ms'],4), round(d['p90_ms'],4), round(d['e2e']['value'],4))" >> gpurun_out/sweep.log
done; done

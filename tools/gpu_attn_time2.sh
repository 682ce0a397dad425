#!/bin/bash
bash tools/gpu_attn_time.sh
timeout 900 python bench.py --model llama-1b --batch 4 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/bench_llama.log 2>&1
python - <<'P'
import json
l=json.loads(open('gpurun_out/bench_llama.log').read().strip().splitlines()[-1])
print('llama', round(l['value']), round(l['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in l['breakdown'].items()})
P

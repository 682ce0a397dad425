#!/bin/bash
# A/B env knobs on the ACCO bench line (no CPU baseline / e2e)
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ab.log 2>&1
  python - "$v" <<'P'
import json,sys
l=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1])
b=l.get('baselines',{})
print(sys.argv[1], 'acco', round(l['value']), round(l['ms_per_step'],3), 'exposed', round(l['exposed_comm_pct'],1), 'zero1', round(b.get('zero1',{}).get('tokens_per_s',0)), 'ddp', round(b.get('ddp',{}).get('tokens_per_s',0)))
P
done

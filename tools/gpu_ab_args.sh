#!/bin/bash
# A/B bench command-line variants (ACCO line only)
for v in "$@"; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines $v > gpurun_out/bench_ab.log 2>&1
  python - "$v" <<'P'
import json,sys
l=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1])
print(repr(sys.argv[1]), round(l['value']), round(l['ms_per_step'],3), 'exposed', round(l['exposed_comm_pct'],1), 'e2e', round(l['e2e']['value']) if l.get('e2e') else None)
P
done

#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_optim.py tests/test_gpu_comm.py tests/test_gpu_peer_world2.py -q -p no:cacheprovider -x > gpurun_out/pytest_bg.log 2>&1
tail -1 gpurun_out/pytest_bg.log; grep -E "^FAILED" gpurun_out/pytest_bg.log | head -3
for v in X=1 ACCO_OPT_FOREGROUND=1; do
for b in 1 8; do
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --batch $b > gpurun_out/bench_bg.log 2>&1
  python - "$v" $b <<'P'
import json,sys
l=json.loads(open('gpurun_out/bench_bg.log').read().strip().splitlines()[-1])
b=l['baselines']
print(sys.argv[1], 'B', sys.argv[2], 'acco', round(l['value']), 'exposed', round(l['exposed_comm_pct'],1), 'zero1', round(b['zero1']['tokens_per_s']), 'speedup', round(l['acco_vs_zero1_speedup'],3), 'e2e', round(l['e2e']['value']))
P
done
done

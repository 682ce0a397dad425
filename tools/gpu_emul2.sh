#!/bin/bash
# ACCO vs ZeRO-1 crossover: smaller micro-batches make the (emulated 8-GPU NVLink) comm a larger share
for b in 1 2 4; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --emulate-comm-gpus 8 --batch $b > gpurun_out/bench_emul8_b$b.log 2>&1
  python - $b <<'P'
import json,sys
l=json.loads(open(f'gpurun_out/bench_emul8_b{sys.argv[1]}.log').read().strip().splitlines()[-1])
b=l['baselines']
print('B', sys.argv[1], 'acco', round(l['value']), 'ms', round(l['ms_per_step'],2), 'exposed', round(l['exposed_comm_pct'],1),
      'zero1', round(b['zero1']['tokens_per_s']), 'ddp', round(b['ddp']['tokens_per_s']), 'speedup', round(l['acco_vs_zero1_speedup'],3))
P
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --batch $b > gpurun_out/bench_b$b.log 2>&1
  python - $b <<'P'
import json,sys
l=json.loads(open(f'gpurun_out/bench_b{sys.argv[1]}.log').read().strip().splitlines()[-1])
b=l['baselines']
print('  no-emul B', sys.argv[1], 'acco', round(l['value']), 'zero1', round(b['zero1']['tokens_per_s']), 'speedup', round(l['acco_vs_zero1_speedup'],3))
P
done

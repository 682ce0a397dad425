#!/bin/bash
# single-GPU overlap study: ACCO vs ZeRO-1 vs DDP with the NVLink time of 2/4/8-GPU collectives emulated
for n in 2 8; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --emulate-comm-gpus $n > gpurun_out/bench_emul$n.log 2>&1
  python - $n <<'P'
import json,sys
l=json.loads(open(f'gpurun_out/bench_emul{sys.argv[1]}.log').read().strip().splitlines()[-1])
b=l['baselines']
print('N', sys.argv[1], 'phase ms', {k: round(v,3) for k,v in l['config']['emulated_interconnect']['phase_ms'].items()},
      'acco', round(l['value']), 'exposed', round(l['exposed_comm_pct'],1),
      'zero1', round(b['zero1']['tokens_per_s']), 'ddp', round(b['ddp']['tokens_per_s']), 'speedup', round(l['acco_vs_zero1_speedup'],3))
P
done

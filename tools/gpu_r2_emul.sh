#!/bin/bash
# ACCO vs ZeRO-1 / DDP under an emulated 8-GPU interconnect on one B200
cd "$(dirname "$0")/.."
for ctas in 0 16 32; do
  python bench.py --steps 15 --warmup 4 --no-cpu-baseline --emulate-comm-gpus 8 --emulate-ctas $ctas 2>&1 | tail -1 | \
  python -c "import sys,json; l=json.loads(sys.stdin.read()); b=l['baselines']; print(json.dumps({'ctas': $ctas, 'acco': round(l['value']), 'zero1': round(b['zero1']['tokens_per_s']), 'ddp': round(b['ddp']['tokens_per_s']), 'acco_vs_zero1': round(l['acco_vs_zero1_speedup'],4), 'acco_vs_ddp': round(l['acco_vs_ddp_speedup'],4), 'exposed_pct': round(l['exposed_comm_pct'],2), 'e2e': round(l['e2e']['value'])}))" | tee -a gpurun_out/r2_emul.jsonl
done

#!/bin/bash
cd "$(dirname "$0")/.."
B="timeout 900 python bench.py --no-cpu-baseline"
show() { python - "$1" "$2" <<'P'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(l['value']), 'acco/zero1', round(l.get('acco_vs_zero1_speedup',0),4), 'zero1', round(l['baselines']['zero1']['tokens_per_s']), 'ddp', round(l['baselines']['ddp']['tokens_per_s']), 'exposed', round(l.get('exposed_comm_pct',0),1), {k:round(v['ms_per_step'],2) for k,v in l['breakdown'].items() if k in ('gemm','attention')})
P
}
for i in 1 2; do
$B --emulate-comm-gpus 8 > gpurun_out/e1.log 2>&1; show gpurun_out/e1.log "emul8"
$B --emulate-comm-gpus 8 --model gpt2-medium > gpurun_out/e2.log 2>&1; show gpurun_out/e2.log "emul8 medium"
done
$B > gpurun_out/e3.log 2>&1; show gpurun_out/e3.log "n1"

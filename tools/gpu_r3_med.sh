#!/bin/bash
cd "$(dirname "$0")/.."
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines"
show() { python - "$1" "$2" <<'P'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(l['value']), round(l['ms_per_step'],3), {k:(round(v['ms_per_step'],3), v['launches_per_step']) for k,v in l['breakdown'].items() if k in ('gemm','layernorm','column_reduce','attention')})
P
}
for i in 1 2; do
$B > gpurun_out/s1.log 2>&1; show gpurun_out/s1.log "small fused"
ACCO_BIAS_COLSUM=1 ACCO_LN_PARAMS_SEPARATE=1 $B > gpurun_out/s2.log 2>&1; show gpurun_out/s2.log "small separate"
$B --model gpt2-medium > gpurun_out/m1.log 2>&1; show gpurun_out/m1.log "medium fused"
ACCO_BIAS_COLSUM=1 ACCO_LN_PARAMS_SEPARATE=1 $B --model gpt2-medium > gpurun_out/m2.log 2>&1; show gpurun_out/m2.log "medium separate"
done

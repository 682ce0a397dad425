#!/bin/bash
cd "$(dirname "$0")/.."
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines"
show() { python - "$1" "$2" <<'P'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(l['value']), round(l['ms_per_step'],3), {k:(round(v['ms_per_step'],3), v['launches_per_step']) for k,v in l['breakdown'].items() if k in ('gemm','layernorm','column_reduce')})
P
}
for i in 1 2; do
$B > gpurun_out/b1.log 2>&1; show gpurun_out/b1.log "all-fused(2/SM)"
ACCO_LN_PART_PER_SM=4 $B > gpurun_out/b2.log 2>&1; show gpurun_out/b2.log "all-fused(4/SM)"
ACCO_LN_PART_PER_SM=8 $B > gpurun_out/b3.log 2>&1; show gpurun_out/b3.log "all-fused(8/SM)"
ACCO_LN_PARAMS_SEPARATE=1 $B > gpurun_out/b4.log 2>&1; show gpurun_out/b4.log "bias-fused,LN-sep"
ACCO_BIAS_COLSUM=1 ACCO_LN_PARAMS_SEPARATE=1 $B > gpurun_out/b5.log 2>&1; show gpurun_out/b5.log "all-separate"
done

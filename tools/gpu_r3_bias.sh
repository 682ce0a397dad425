#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_b1.csv python bench.py --steps 2 --warmup 1 --profile --no-baselines --no-cpu-baseline > /dev/null 2>&1
ACCO_BIAS_COLSUM=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_b0.csv python bench.py --steps 2 --warmup 1 --profile --no-baselines --no-cpu-baseline > /dev/null 2>&1
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines"
show() { python - "$1" "$2" <<'P'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(l['value']), round(l['ms_per_step'],3), {k:(round(v['ms_per_step'],3), v['launches_per_step']) for k,v in l['breakdown'].items() if k in ('gemm','layernorm','column_reduce','attention')})
P
}
for i in 1 2 3; do
$B > gpurun_out/s1.log 2>&1; show gpurun_out/s1.log "bias-mma"
ACCO_BIAS_COLSUM=1 $B > gpurun_out/s2.log 2>&1; show gpurun_out/s2.log "bias-colsum"
done

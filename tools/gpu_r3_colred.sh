#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest -q -m gpu tests/test_gpu_model.py -x -k "fused_bias or wide_row or bench" > gpurun_out/colred_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/colred_pytest.log; tail -3 gpurun_out/colred_pytest.log; grep -E "Error|assert" gpurun_out/colred_pytest.log | head -5
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines"
for i in 1 2; do
$B > gpurun_out/b_new.log 2>&1; python - <<'P'
import json
l=json.loads(open('gpurun_out/b_new.log').read().strip().splitlines()[-1])
print('fused', round(l['value']), round(l['ms_per_step'],3), {k:(round(v['ms_per_step'],3), v['launches_per_step']) for k,v in l['breakdown'].items()})
P
ACCO_BIAS_COLSUM=1 ACCO_LN_PARAMS_SEPARATE=1 $B > gpurun_out/b_old.log 2>&1; python - <<'P'
import json
l=json.loads(open('gpurun_out/b_old.log').read().strip().splitlines()[-1])
print('separate', round(l['value']), round(l['ms_per_step'],3), {k:(round(v['ms_per_step'],3), v['launches_per_step']) for k,v in l['breakdown'].items()})
P
done

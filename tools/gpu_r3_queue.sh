#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_llama.py -q -x > gpurun_out/q_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/q_pytest.log; tail -2 gpurun_out/q_pytest.log
timeout 300 python tools/diag/gemm_cfg_time.py 8192 2304 768 0 0 store auto 256,1,2 256,1
timeout 300 python tools/diag/gemm_cfg_time.py 8192 50257 768 0 0 store auto 256,1
B="timeout 900 python bench.py --no-cpu-baseline"
show() { python - "$1" "$2" <<'P'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], round(l['value']), 'acco/zero1', round(l.get('acco_vs_zero1_speedup',0),4), 'zero1', round(l['baselines']['zero1']['tokens_per_s']), 'exposed', round(l.get('exposed_comm_pct',0),1), 'gemm frac', round(l['roofline']['frac'],3))
P
}
$B --emulate-comm-gpus 8 > gpurun_out/e1.log 2>&1; show gpurun_out/e1.log "emul8 queue"
ACCO_GEMM_NO_CG2=1 $B --emulate-comm-gpus 8 > gpurun_out/e2.log 2>&1; show gpurun_out/e2.log "emul8 no-cg2"
$B > gpurun_out/e3.log 2>&1; show gpurun_out/e3.log "n1 queue"

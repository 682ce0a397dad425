#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_model.py tests/test_gpu_llama.py tests/test_gpu_bench_shapes.py > gpurun_out/attn_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/attn_pytest.log; grep -E "passed|failed|FAILED" gpurun_out/attn_pytest.log | tail -5
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines"
$B > gpurun_out/b_s.log 2>&1; python - <<'P'
import json
l=json.loads(open('gpurun_out/b_s.log').read().strip().splitlines()[-1])
print(round(l['value']), round(l['ms_per_step'],3), 'gemm frac', round(l['roofline']['frac'],3), 'attn', round(l['attention']['tflops']), {k:round(v['ms_per_step'],3) for k,v in l['breakdown'].items()})
P

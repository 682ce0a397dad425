#!/bin/bash
# quick loop: GPU model/attention parity tests + a short bench (breakdown printed)
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_llama.py tests/test_gpu_engine.py -q -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1
tail -3 gpurun_out/pytest_quick.log; grep -E "^FAILED|Error" gpurun_out/pytest_quick.log | head -5
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines ${BENCH_ARGS} > gpurun_out/bench_quick.log 2>&1
python - <<'P'
import json
l=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1])
print(round(l['value']), round(l['ms_per_step'],3), 'gemm frac', round(l['roofline']['frac'],3), 'attn', round(l['attention']['tflops']), {k:round(v['ms_per_step'],3) for k,v in l['breakdown'].items()})
P

#!/bin/bash
# A/B of an env knob on the bench (breakdown printed), after the GPU test suite
timeout 1200 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head -5
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_ab.log 2>&1
  python - "$v" <<'P'
import json,sys
l=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1])
print(sys.argv[1], round(l['value']), round(l['ms_per_step'],3), 'gemm frac', round(l['roofline']['frac'],3), 'attn', round(l['attention']['tflops']), {k:round(v['ms_per_step'],3) for k,v in l['breakdown'].items()})
P
done

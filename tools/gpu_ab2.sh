#!/bin/bash
# quick parity tests, then A/B env knobs on the ACCO bench line (breakdown)
timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_engine.py -q -p no:cacheprovider -x > gpurun_out/pytest_ab.log 2>&1
tail -1 gpurun_out/pytest_ab.log; grep -E "^FAILED" gpurun_out/pytest_ab.log | head -3
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_ab.log 2>&1
  python - "$v" <<'P'
import json,sys
l=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1])
print(sys.argv[1], round(l['value']), round(l['ms_per_step'],3), 'gemm', round(l['roofline']['frac'],3), {k:round(v['ms_per_step'],2) for k,v in l['breakdown'].items()})
P
done

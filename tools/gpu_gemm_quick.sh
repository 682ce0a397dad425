#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py -q -p no:cacheprovider -x > gpurun_out/pytest_gemm.log 2>&1
tail -2 gpurun_out/pytest_gemm.log; grep -E "^FAILED|Error" gpurun_out/pytest_gemm.log | head -5
timeout 300 python tools/gemm_bench.py 768 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    if 'name' in d: print(f\"{d['name']:12s} {d['ms']*1000:7.1f}us {d['tflops']:7.1f}\")
    else: print(d)"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_quick.log 2>&1
python - <<'P'
import json
l=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1])
print(round(l['value']), round(l['ms_per_step'],3), 'gemm frac', round(l['roofline']['frac'],3), 'attn', round(l['attention']['tflops']), {k:round(v['ms_per_step'],3) for k,v in l['breakdown'].items()})
P

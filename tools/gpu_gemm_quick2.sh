#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py tests/test_gpu_llama.py tests/test_gpu_engine.py -q -p no:cacheprovider -x > gpurun_out/pytest_gemm.log 2>&1
tail -1 gpurun_out/pytest_gemm.log; grep -E "^FAILED|^E  " gpurun_out/pytest_gemm.log | head -5
timeout 300 python tools/gemm_bench.py 768 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    if 'name' in d: print(f\"{d['name']:16s} {d['ms']*1000:7.1f}us {d['tflops']:7.1f}\")
    else: print(d)"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_quick.log 2>&1
python -c "import json; l=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1]); print(round(l['value']), round(l['ms_per_step'],3), 'gemm', round(l['roofline']['frac'],3), {k:round(v['ms_per_step'],2) for k,v in l['breakdown'].items()})"
timeout 900 python bench.py --model llama-1b --batch 4 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/bl.log 2>&1
python -c "import json; l=json.loads(open('gpurun_out/bl.log').read().strip().splitlines()[-1]); print('llama', round(l['value']), round(l['ms_per_step'],2), {k:round(v['ms_per_step'],2) for k,v in l['breakdown'].items()})"

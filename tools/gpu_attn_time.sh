#!/bin/bash
# attention kernel times (ncu, serialized) + quick parity tests + bench
timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_llama.py -q -p no:cacheprovider -x > gpurun_out/pytest_attn.log 2>&1
tail -2 gpurun_out/pytest_attn.log; grep -E "^FAILED|Error" gpurun_out/pytest_attn.log | head -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_|dsum" -s 8 -c 8 --csv python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline 2>/dev/null | grep -E "fa_|dsum" | awk -F'","' '{split($5,a,"("); n[a[1]]++; t[a[1]]+=$NF} END {for (k in n) print k, t[k]/n[k]/1000, "us"}'
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_quick.log 2>&1
python - <<'P'
import json
l=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1])
print(round(l['value']), round(l['ms_per_step'],3), 'gemm frac', round(l['roofline']['frac'],3), 'attn', round(l['attention']['tflops']), {k:round(v['ms_per_step'],3) for k,v in l['breakdown'].items()})
P

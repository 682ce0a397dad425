#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_model.py tests/test_gpu_llama.py tests/test_gpu_bench_shapes.py tests/test_gpu_engine.py -q -m gpu -x 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>&1 | tail -1 | cut -c1-160
for emu in "" "--emulate-comm-gpus 8 --emulate-ctas 16"; do
  python bench.py --model gpt2-medium --steps 8 --warmup 3 --no-cpu-baseline $emu 2>&1 | tail -1 | \
  python -c "import sys,json; l=json.loads(sys.stdin.read()); b=l['baselines']; print(json.dumps({'model': 'gpt2-medium', 'emu': '$emu', 'acco': round(l['value']), 'zero1': round(b['zero1']['tokens_per_s']), 'ddp': round(b['ddp']['tokens_per_s']), 'acco_vs_zero1': round(l['acco_vs_zero1_speedup'],4), 'exposed_pct': round(l['exposed_comm_pct'],2), 'gemm_frac': round(l['roofline']['frac'],4)}))"
done

#!/bin/bash
# CLC GEMM: correctness (GEMM + model tests), then A/B vs the static schedule, plain and under emulated comm
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py tests/test_gpu_bench_shapes.py -x -q -m gpu 2>&1 | tail -3
for knob in "" "ACCO_GEMM_NO_CLC=1"; do
  for emu in "" "--emulate-comm-gpus 8 --emulate-ctas 16"; do
    env $knob python bench.py --steps 15 --warmup 4 --no-cpu-baseline $emu 2>&1 | tail -1 | \
    python -c "import sys,json; l=json.loads(sys.stdin.read()); b=l['baselines']; print(json.dumps({'knob': '$knob', 'emu': '$emu', 'acco': round(l['value']), 'zero1': round(b['zero1']['tokens_per_s']), 'ddp': round(b['ddp']['tokens_per_s']), 'acco_vs_zero1': round(l['acco_vs_zero1_speedup'],4), 'exposed_pct': round(l['exposed_comm_pct'],2), 'gemm_frac': round(l['roofline']['frac'],4)}))"
  done
done

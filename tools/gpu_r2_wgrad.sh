#!/bin/bash
# weight-gradient GEMMs on the side stream (with CLC) vs inline: correctness, then interleaved A/B
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_bench_shapes.py tests/test_gpu_engine.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do
for knob in "" "ACCO_WGRAD_INLINE=1" "ACCO_WGRAD_INLINE=1 ACCO_GEMM_NO_CLC=1"; do
  env $knob python bench.py --steps 15 --warmup 4 --no-cpu-baseline --no-baselines 2>&1 | tail -1 | \
  python -c "import sys,json; l=json.loads(sys.stdin.read()); print('$knob', round(l['value']), round(l['ms_per_step'],3), round(l['roofline']['frac'],4))"
done; done

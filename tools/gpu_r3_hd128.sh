#!/bin/bash
# Head size 128 on the tcgen05 attention kernels: parity tests, the hd=64
# attention regression, hd=128 timings, and the bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_head128.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_llama.py -x -q 2>&1 | tail -5
for a in "8 1024 12 12 20 64" "4 2048 32 4 10 64" "8 1024 6 6 20 128" "4 2048 16 16 10 128" "4 2048 32 8 10 128" "1 8192 32 8 5 128"; do
  timeout 120 tools/diag/attn_bench.bin $a
done | tee gpurun_out/hd128_attn.jsonl
timeout 300 python bench.py --steps 10 --warmup 3 2>&1 | tail -1

#!/bin/bash
# dK/dV lse / D as bulk copies (T % 4 == 0) or per-lane 4 B copies: timing + attention parity tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
  echo "old $r"; tools/diag/attn_bench_old.bin 8 1024 12 12 20 | tail -1
  echo "new $r"; tools/diag/attn_bench.bin 8 1024 12 12 20 | tail -1
done
echo "new T=1022 (per-lane path)"; tools/diag/attn_bench.bin 8 1022 12 12 20 | tail -1
echo "old gqa"; tools/diag/attn_bench_old.bin 4 2048 32 4 10 | tail -1
echo "new gqa"; tools/diag/attn_bench.bin 4 2048 32 4 10 | tail -1
echo "old hd128"; tools/diag/attn_bench_old.bin 4 2048 16 16 10 128 | tail -1
echo "new hd128"; tools/diag/attn_bench.bin 4 2048 16 16 10 128 | tail -1
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_model.py tests/test_gpu_llama.py tests/test_gpu_bench_shapes.py tests/test_gpu_head128.py > gpurun_out/attn_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/attn_pytest.log; grep -E "passed|failed|FAILED|rc=" gpurun_out/attn_pytest.log | tail -5

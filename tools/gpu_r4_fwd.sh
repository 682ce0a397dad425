#!/bin/bash
# forward with one MMA issuer per tile slot: A/B timing vs the previous commit, probe timeline, attention parity tests, one bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
  echo "base $r"; timeout 60 tools/diag/attn_bench_base.bin 8 1024 12 12 20 | tail -1
  echo "new $r"; timeout 60 tools/diag/attn_bench.bin 8 1024 12 12 20 | tail -1
done
echo "base gqa"; timeout 60 tools/diag/attn_bench_base.bin 4 2048 32 4 10 | tail -1
echo "new gqa"; timeout 60 tools/diag/attn_bench.bin 4 2048 32 4 10 | tail -1
echo "base hd128"; timeout 60 tools/diag/attn_bench_base.bin 4 2048 16 16 10 128 | tail -1
echo "new hd128"; timeout 60 tools/diag/attn_bench.bin 4 2048 16 16 10 128 | tail -1
echo "new T=1022 / odd tile count T=900"; timeout 60 tools/diag/attn_bench.bin 8 1022 12 12 5 | tail -1; timeout 60 tools/diag/attn_bench.bin 8 900 12 12 5 | tail -1
timeout 60 tools/diag/fwd_probe.bin 2>&1 | tail -20
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_model.py tests/test_gpu_llama.py tests/test_gpu_bench_shapes.py tests/test_gpu_head128.py > gpurun_out/attn_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/attn_pytest.log; grep -E "passed|failed|FAILED|rc=" gpurun_out/attn_pytest.log | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/b_s3.log 2>&1; tail -1 gpurun_out/b_s3.log | cut -c1-200

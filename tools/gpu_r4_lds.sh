#!/bin/bash
# shared-space smem pointers (LDS/STS instead of generic LD/ST) in the GEMM and attention kernels:
# attention A/B, bench A/B against the previous commit's build (_old), full GPU suite
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
  echo "base $r"; timeout 60 tools/diag/attn_bench_base.bin 8 1024 12 12 20 | tail -1
  echo "new $r"; timeout 60 tools/diag/attn_bench.bin 8 1024 12 12 20 | tail -1
done
echo "base gqa"; timeout 60 tools/diag/attn_bench_base.bin 4 2048 32 4 10 | tail -1
echo "new gqa"; timeout 60 tools/diag/attn_bench.bin 4 2048 32 4 10 | tail -1
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines"
for r in 1 2; do
  (cd _old && $B > ../gpurun_out/b_old$r.log 2>&1); echo "old $(python -c "import json;l=json.loads(open('gpurun_out/b_old$r.log').read().strip().splitlines()[-1]);print(round(l['value']),l['clocks']['sm_mhz'],round(l['roofline']['frac'],3),round(l['attention']['tflops']))")"
  $B > gpurun_out/b_new$r.log 2>&1; echo "new $(python -c "import json;l=json.loads(open('gpurun_out/b_new$r.log').read().strip().splitlines()[-1]);print(round(l['value']),l['clocks']['sm_mhz'],round(l['roofline']['frac'],3),round(l['attention']['tflops']))")"
done
(cd _old && timeout 600 python bench.py --model llama-1b --batch 4 --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > ../gpurun_out/bl_old.log 2>&1); echo "llama old $(tail -1 gpurun_out/bl_old.log | cut -c1-70)"
timeout 600 python bench.py --model llama-1b --batch 4 --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bl_new.log 2>&1; echo "llama new $(tail -1 gpurun_out/bl_new.log | cut -c1-70)"
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/full_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/full_pytest.log | tail -3

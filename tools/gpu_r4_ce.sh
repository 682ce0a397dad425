#!/bin/bash
# cross-entropy row staged in shared memory (one HBM read + one write per logit) vs the L2 re-read (ACCO_CE_NO_SMEM)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines"
show() { python -c "import json;l=json.loads(open('$1').read().strip().splitlines()[-1]);b=l.get('breakdown',{});print(round(l['value']),l['clocks']['sm_mhz'],{k:round(v['ms_per_step'],3) for k,v in b.items() if k in ('cross_entropy','ce','loss')} or list(b)[:12])"; }
for r in 1 2; do
  ACCO_CE_NO_SMEM=1 $B > gpurun_out/b_ce_old$r.log 2>&1; echo "old $(show gpurun_out/b_ce_old$r.log)"
  $B > gpurun_out/b_ce_new$r.log 2>&1; echo "new $(show gpurun_out/b_ce_new$r.log)"
done
N="ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ce_vec -c 2 --csv"
ACCO_CE_NO_SMEM=1 timeout 300 $N python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-baselines 2>/dev/null | grep -E "ce_vec" | cut -c1-50,150-400 | tail -6
timeout 300 $N python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-baselines 2>/dev/null | grep -E "ce_vec" | cut -c1-50,150-400 | tail -6
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_model.py tests/test_gpu_bench_shapes.py tests/test_gpu_llama.py tests/test_gpu_engine.py > gpurun_out/ce_pytest.log 2>&1; echo "rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/ce_pytest.log | tail -3

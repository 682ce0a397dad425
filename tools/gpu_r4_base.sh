#!/bin/bash
# session start on a rebuilt tree: attention timing, full GPU suite + smoke, one bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tools/diag/attn_bench.bin 8 1024 12 12 20 > gpurun_out/attn_base.log 2>&1; cat gpurun_out/attn_base.log | tail -6
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/full_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/full_pytest.log
grep -E "passed|failed|FAILED|Error" gpurun_out/full_pytest.log | tail -8
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/b_s.log 2>&1; tail -1 gpurun_out/b_s.log | cut -c1-300

#!/bin/bash
# full GPU suite + smoke, then a few bench A/Bs
cd "$(dirname "$0")/.."
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/full_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/full_pytest.log
grep -E "passed|failed|FAILED|Error" gpurun_out/full_pytest.log | tail -8
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines"
$B --model llama-1b --batch 4 > gpurun_out/b_l.log 2>&1; echo "llama $(tail -1 gpurun_out/b_l.log | cut -c1-80)"
ACCO_DSWIGLU_CG2=1 $B --model llama-1b --batch 4 > gpurun_out/b_l2.log 2>&1; echo "llama dswiglu-cg2 $(tail -1 gpurun_out/b_l2.log | cut -c1-80)"

#!/bin/bash
# full GPU suite + smoke (round-2 regression check)
cd "$(dirname "$0")/.."
python tools/diag/tf32_accuracy.py > gpurun_out/tf32_acc.jsonl 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_full_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_full_pytest.log
grep -E "passed|failed|FAILED|Error" gpurun_out/r2_full_pytest.log | tail -25
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3

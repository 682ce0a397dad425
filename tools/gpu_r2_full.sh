#!/bin/bash
# full GPU suite + smoke (round-2 regression check)
cd "$(dirname "$0")/.."
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r2_full_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_full_pytest.log
tail -15 gpurun_out/r2_full_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3

#!/bin/bash
# baseline of the restored tree: GPU suite + smoke + default bench
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/base_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/base_pytest.log
tail -5 gpurun_out/base_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/base_bench.log 2>&1; tail -1 gpurun_out/base_bench.log

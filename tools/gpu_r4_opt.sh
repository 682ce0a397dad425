#!/bin/bash
# AdamW kernels on an occupancy-sized grid vs the old fixed 8 x 148 grid: microbench, optimizer tests, bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
  echo "occupancy grid $r"; timeout 300 python tools/optim_microbench.py --sizes 1.244e8,1e9 --reps 10 2>&1 | grep -v "^\[" | cut -c1-400 | tail -2
  echo "fixed 1184 $r"; ACCO_OPT_BLOCKS=1184 timeout 300 python tools/optim_microbench.py --sizes 1.244e8,1e9 --reps 10 2>&1 | cut -c1-400 | tail -2
done
timeout 900 python -m pytest -q -m gpu tests/test_gpu_optim.py tests/test_gpu_engine.py tests/test_gpu_comm.py > gpurun_out/opt_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/opt_pytest.log; grep -E "passed|failed|FAILED|rc=" gpurun_out/opt_pytest.log | tail -4
for r in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/b_o.log 2>&1; echo "new $(tail -1 gpurun_out/b_o.log | cut -c1-120)"
ACCO_OPT_BLOCKS=1184 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/b_o2.log 2>&1; echo "old $(tail -1 gpurun_out/b_o2.log | cut -c1-120)"
done

#!/bin/bash
# Llama (C4) GPU check: parity tests, the full GPU suite (regressions), and a llama-1b bench line.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -m pytest tests/test_gpu_llama.py -q -p no:cacheprovider -x > gpurun_out/pytest_llama.log 2>&1
tail -15 gpurun_out/pytest_llama.log
timeout 1200 python -m pytest tests/ -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
timeout 600 python bench.py --model llama-1b --batch 4 --steps 5 --warmup 3 --no-baselines > gpurun_out/bench_llama.log 2>&1
tail -2 gpurun_out/bench_llama.log | cut -c1-1500
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_quick.log 2>&1
tail -1 gpurun_out/bench_quick.log | cut -c1-300

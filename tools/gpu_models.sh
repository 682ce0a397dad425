#!/bin/bash
# bench lines for the other configs (C3 GPT-2 medium, C4 Llama-style 1.1B, C1 tiny)
timeout 600 python bench.py --model gpt2-medium --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gpt2m.log 2>&1; tail -1 gpurun_out/bench_gpt2m.log | cut -c1-200
timeout 900 python bench.py --model llama-1b --batch 4 --steps 5 --warmup 3 > gpurun_out/bench_llama.log 2>&1; tail -1 gpurun_out/bench_llama.log | cut -c1-200
timeout 300 python bench.py --model c1 --batch 8 --steps 20 --warmup 3 > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log | cut -c1-200

#!/bin/bash
# final bench lines of the session (N = 1): default, GPT-2 medium, Llama-1B, reference arm
cd "$(dirname "$0")/.."
timeout 900 python bench.py > gpurun_out/r02_bench_final.log 2>&1; tail -1 gpurun_out/r02_bench_final.log | cut -c1-200
timeout 900 python bench.py --model gpt2-medium --no-cpu-baseline > gpurun_out/r02_bench_gpt2_medium.log 2>&1; tail -1 gpurun_out/r02_bench_gpt2_medium.log | cut -c1-120
timeout 900 python bench.py --model llama-1b --batch 4 --no-cpu-baseline > gpurun_out/r02_bench_llama_1b.log 2>&1; tail -1 gpurun_out/r02_bench_llama_1b.log | cut -c1-120
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference_arm.log 2>&1; tail -1 gpurun_out/r02_bench_reference_arm.log | cut -c1-160
timeout 900 python bench.py --emulate-comm-gpus 8 --no-cpu-baseline > gpurun_out/r02_bench_emul8.log 2>&1; tail -1 gpurun_out/r02_bench_emul8.log | cut -c1-120

#!/bin/bash
# End-of-round evidence in one call: GPU suite, smoke, bench (both arms), other
# model configs, launch list, and full ncu captures of every hot kernel class.
bash tools/gpu_round.sh
timeout 600 python bench.py --model llama-1b --batch 4 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/bench_llama.log 2>&1; tail -1 gpurun_out/bench_llama.log | cut -c1-300
timeout 600 python bench.py --model gpt2-medium --steps 5 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/bench_gpt2_medium.log 2>&1; tail -1 gpurun_out/bench_gpt2_medium.log | cut -c1-300
P="python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:gemm_tc_kernel -s 60 -c 12 -o gpurun_out/prof_gemm $P > gpurun_out/ncu_gemm.log 2>&1
timeout 900 $N -k regex:"fa_bwd|fa_fwd" -s 24 -c 3 -o gpurun_out/prof_attn $P > gpurun_out/ncu_attn.log 2>&1
timeout 900 $N -k regex:"opt_kernel|ce_vec" -c 3 -o gpurun_out/prof_opt_ce $P > gpurun_out/ncu_opt.log 2>&1
ls -la gpurun_out/*.ncu-rep

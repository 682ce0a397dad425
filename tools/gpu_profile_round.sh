#!/bin/bash
# Round profile evidence: bench line, launch list of a bench step, and full ncu
# captures of every hot kernel class (GEMM fwd/dgrad/wgrad, attention fwd/dq/dkv,
# fused AdamW estimate/commit, cross-entropy).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1
tail -1 gpurun_out/bench_full.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --profile --no-baselines --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
P="python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:gemm_tc_kernel -s 60 -c 12 -o gpurun_out/prof_gemm $P > gpurun_out/ncu_gemm.log 2>&1
timeout 900 $N -k regex:"fa_bwd|fa_fwd" -s 24 -c 3 -o gpurun_out/prof_attn $P > gpurun_out/ncu_attn.log 2>&1
timeout 900 $N -k regex:"opt_kernel|ce_vec" -c 3 -o gpurun_out/prof_opt_ce $P > gpurun_out/ncu_opt.log 2>&1
ls -la gpurun_out/*.ncu-rep

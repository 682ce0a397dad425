#!/bin/bash
# Round-2 profile evidence: launch list of a bench step and ncu --set full captures of every hot kernel class
# (GEMM fwd/dgrad/wgrad incl. CLC, attention fwd/dq/dkv, fused AdamW, cross-entropy, the 3xTF32 fp32 GEMM).
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --profile --no-baselines --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
P="python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:gemm_tc_kernel -s 60 -c 12 -o gpurun_out/r02_prof_gemm $P > gpurun_out/ncu_gemm.log 2>&1
timeout 900 $N -k regex:"fa_bwd|fa_fwd" -s 24 -c 3 -o gpurun_out/r02_prof_attn $P > gpurun_out/ncu_attn.log 2>&1
timeout 900 $N -k regex:"opt_kernel|ce_vec" -c 3 -o gpurun_out/r02_prof_opt_ce $P > gpurun_out/ncu_opt.log 2>&1
timeout 900 $N -k regex:"gemm_tc_kernel|tf32_split" -c 6 -o gpurun_out/r02_prof_tf32 python tools/diag/tf32_accuracy.py > gpurun_out/ncu_tf32.log 2>&1
ls -la gpurun_out/*.ncu-rep

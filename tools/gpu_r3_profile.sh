#!/bin/bash
# End-of-session profile evidence on the final tree: launch list of a bench step
# and ncu --set full captures of the hot kernel classes (GEMM incl. CTA-pair
# tiles, attention fwd/dq/dkv, fused AdamW, CE, fused norm backward).
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
[ -n "$SKIP_LAUNCHES" ] || timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --profile --no-baselines --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
P="python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on"
# the last layer's forward (qkv / fc on CTA-pair tiles, proj / fc2), the LM head (forward and weight gradient
# on pair tiles, dgrad as fp32-workspace split-K) and the last layer's backward (weight gradients with the
# fused bias gradient)
timeout 900 $N -k regex:gemm_tc_kernel -s 44 -c 15 -o gpurun_out/r02_prof_gemm $P > gpurun_out/ncu_gemm.log 2>&1
timeout 900 $N -k regex:"fa_bwd|fa_fwd" -s 24 -c 3 -o gpurun_out/r02_prof_attn $P > gpurun_out/ncu_attn.log 2>&1
timeout 900 $N -k regex:"fa_fwd" -s 1 -c 2 -o gpurun_out/r02_prof_attnf $P > gpurun_out/ncu_attnf.log 2>&1
timeout 900 $N -k regex:"opt_kernel" -c 2 -o gpurun_out/r02_prof_opt $P > gpurun_out/ncu_opt.log 2>&1
timeout 900 $N -k regex:"ce_vec|ln_bwd_vec_p" -c 5 -o gpurun_out/r02_prof_ce_ln $P > gpurun_out/ncu_ce.log 2>&1
timeout 900 $N -k regex:"ln_param_fold|ln_fwd_vec" -c 3 -o gpurun_out/r02_prof_misc $P > gpurun_out/ncu_misc.log 2>&1
ls -la gpurun_out/*.ncu-rep

#!/bin/bash
cd "$(dirname "$0")/.."
P="python bench.py --steps 1 --warmup 1 --no-baselines --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ln_bwd_vec" -s 10 -c 2 -o gpurun_out/ln_fused $P > /dev/null 2>&1
ACCO_LN_PARAMS_SEPARATE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ln_bwd_vec" -s 10 -c 2 -o gpurun_out/ln_sep $P > /dev/null 2>&1
ls -la gpurun_out/ln_*.ncu-rep

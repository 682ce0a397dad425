#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fa_" -s 12 -c 3 -o gpurun_out/prof_attn2 python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline > gpurun_out/ncu_attn2.log 2>&1
tail -2 gpurun_out/ncu_attn2.log

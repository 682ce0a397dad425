#!/bin/bash
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_llama.csv python bench.py --model llama-1b --batch 4 --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline > gpurun_out/llama_ncu.log 2>&1
tail -1 gpurun_out/llama_ncu.log | cut -c1-100

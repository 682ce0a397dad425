#!/bin/bash
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
(nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 500 > gpurun_out/gemm_model_clocks.csv &) 
ACCO_GEMM_LOG=1 timeout 1500 python tools/diag/gemm_model_check.py > gpurun_out/gemm_model2.jsonl 2> gpurun_out/gemm_model2.err
tail -2 gpurun_out/gemm_model2.err; wc -l gpurun_out/gemm_model2.jsonl

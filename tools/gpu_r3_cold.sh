#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python tools/diag/gemm_cold.py 2>&1 | tee gpurun_out/gemm_cold.jsonl | tail -2

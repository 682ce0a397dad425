#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/diag/gemm_pdl_check.py 2>&1 | tee gpurun_out/pdl_check.jsonl
ACCO_NO_PDL=1 timeout 300 python tools/diag/gemm_pdl_check.py 2>&1 | tee -a gpurun_out/pdl_check.jsonl

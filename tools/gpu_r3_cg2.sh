#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python tools/diag/gemm_cg2_check.py > gpurun_out/cg2.jsonl 2>&1
echo "rc=$?" >> gpurun_out/cg2.jsonl
tail -30 gpurun_out/cg2.jsonl

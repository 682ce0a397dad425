#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ACCO_NO_PDL=1 TAG=nopdl timeout 300 python tools/diag/gemm_insitu.py > gpurun_out/insitu_nopdl.json 2>gpurun_out/insitu.err
ACCO_GEMM_LOG=1 ACCO_NO_PDL=1 timeout 300 python tools/diag/gemm_insitu.py 2>&1 >/dev/null | grep "^gemm" > gpurun_out/insitu_plans.txt
tail -3 gpurun_out/insitu.err

#!/bin/bash
cd "$(dirname "$0")/.."
N="ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 4 -c 1"
ACCO_GEMM_FORCE=192,1 timeout 300 $N -o gpurun_out/g_proj192 python tools/diag/gemm_cfg_time.py 8192 768 768 0 0 store auto > /dev/null 2>&1
ACCO_GEMM_FORCE=256,1,2 timeout 300 $N -o gpurun_out/g_qkv256p python tools/diag/gemm_cfg_time.py 8192 2304 768 0 0 store auto > /dev/null 2>&1
ACCO_GEMM_FORCE=192,1 timeout 300 $N -o gpurun_out/g_qkv192 python tools/diag/gemm_cfg_time.py 8192 2304 768 0 0 store auto > /dev/null 2>&1
ls gpurun_out/g_*.ncu-rep

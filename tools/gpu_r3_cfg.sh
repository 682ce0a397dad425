#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python tools/diag/gemm_cg2_check.py 2>&1 | grep -v '"ok": true' | head -20
T="timeout 300 python tools/diag/gemm_cfg_time.py"
{
$T 8192 768 768 0 0 store auto 192,1 256,1,2 192,1,2 128,1,2
$T 8192 768 3072 0 0 store auto 192,1 256,1,2 192,1,2 128,1,2
$T 8192 2304 768 0 0 store auto 256,1 256,1,2 192,1,2 128,1,2
$T 8192 3072 768 0 0 gelu auto 256,1,2 192,1,2 128,1,2
$T 8192 3072 768 0 1 dgelu auto 256,1,2 128,1,2
$T 8192 768 3072 0 1 store auto 256,1,2 128,1,2
$T 8192 768 768 0 1 store auto 256,1,2 128,1,2
$T 768 3072 8192 1 1 acc_f32 auto 128,1,2
$T 2304 768 8192 1 1 acc_f32 auto 128,1,2
$T 50257 768 8192 1 1 acc_f32 auto 256,1,2
$T 8192 50257 768 0 0 store auto 256,1,2
} > gpurun_out/cfg2.jsonl 2>&1
cat gpurun_out/cfg2.jsonl

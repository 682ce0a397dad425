#!/bin/bash
# A/B of the CTA-pair GEMM tiles on the three bench models (same box, interleaved)
cd "$(dirname "$0")/.."
B="timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines"
for i in 1 2; do
  $B > gpurun_out/b_s.log 2>&1; echo "small cg2 $(tail -1 gpurun_out/b_s.log | cut -c1-80)"
  ACCO_GEMM_NO_CG2=1 $B > gpurun_out/b_s0.log 2>&1; echo "small cg1 $(tail -1 gpurun_out/b_s0.log | cut -c1-80)"
done
$B --model gpt2-medium > gpurun_out/b_m.log 2>&1; echo "medium cg2 $(tail -1 gpurun_out/b_m.log | cut -c1-80)"
ACCO_GEMM_NO_CG2=1 $B --model gpt2-medium > gpurun_out/b_m0.log 2>&1; echo "medium cg1 $(tail -1 gpurun_out/b_m0.log | cut -c1-80)"
$B --model llama-1b --batch 4 > gpurun_out/b_l.log 2>&1; echo "llama cg2 $(tail -1 gpurun_out/b_l.log | cut -c1-80)"
ACCO_SWIGLU_CG2=1 $B --model llama-1b --batch 4 > gpurun_out/b_l2.log 2>&1; echo "llama cg2+swiglu $(tail -1 gpurun_out/b_l2.log | cut -c1-80)"
ACCO_GEMM_NO_CG2=1 $B --model llama-1b --batch 4 > gpurun_out/b_l0.log 2>&1; echo "llama cg1 $(tail -1 gpurun_out/b_l0.log | cut -c1-80)"

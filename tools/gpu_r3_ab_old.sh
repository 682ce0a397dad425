#!/bin/bash
# GEMM tile-config times: the _ab_old worktree vs this tree, same box, alternating
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
  timeout 600 python _ab_old/tools/diag/gemm_model_check.py gpt2-small 2>/dev/null | sed 's/^/old /' | head -${NSH:-5}
  timeout 600 python tools/diag/gemm_model_check.py gpt2-small 2>/dev/null | sed 's/^/new /' | head -${NSH:-5}
done > gpurun_out/ab_old.txt 2>&1

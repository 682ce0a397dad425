#!/bin/bash
# What bounds the dK/dV tile: full kernel vs no softmax math vs no TMEM traffic either (diagnostic builds)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for b in attn_bench attn_bench_dacco_diag_dkv_no_math attn_bench_dacco_diag_dkv_no_mathdacco_diag_dkv_no_tmem; do
  echo "== $b"
  timeout 120 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_uniform.avg --cache-control none --clock-control none -k regex:"fa_bwd|fa_fwd" -s 6 -c 3 tools/diag/$b.bin 8 1024 12 12 3 64 2>&1 | grep -E "fa_|duration|pct|uniform" | sed 's/  */ /g'
done

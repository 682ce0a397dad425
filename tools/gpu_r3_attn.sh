#!/bin/bash
cd "$(dirname "$0")/.."
tools/diag/attn_bench.bin 8 1024 12 12 20
tools/diag/attn_bench.bin 4 2048 32 4 10
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:"fa_bwd_dkv" -s 3 -c 1 -o gpurun_out/attn_dkv tools/diag/attn_bench.bin 8 1024 12 12 1 > /dev/null 2>&1
timeout 600 $N -k regex:"fa_fwd_tc2" -s 3 -c 1 -o gpurun_out/attn_fwd tools/diag/attn_bench.bin 8 1024 12 12 1 > /dev/null 2>&1
timeout 600 $N -k regex:"fa_bwd_dq" -s 3 -c 1 -o gpurun_out/attn_dq tools/diag/attn_bench.bin 8 1024 12 12 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep

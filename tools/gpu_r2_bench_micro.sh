#!/bin/bash
cd "$(dirname "$0")/.."
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.log 2>&1; tail -1 gpurun_out/r2_bench.log | cut -c1-3000
python tools/optim_microbench.py --sizes 1e7,1e8,1e9 --reps 10 > gpurun_out/r2_micro_nccl.jsonl 2>&1; tail -3 gpurun_out/r2_micro_nccl.jsonl
python tools/optim_microbench.py --fabric peer --sizes 1e7,1e8 --reps 6 > gpurun_out/r2_micro_peer.jsonl 2>&1; tail -2 gpurun_out/r2_micro_peer.jsonl

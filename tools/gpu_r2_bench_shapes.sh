#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests/test_gpu_bench_shapes.py -x -q -s -m gpu > gpurun_out/r2_bench_shapes.log 2>&1
tail -80 gpurun_out/r2_bench_shapes.log

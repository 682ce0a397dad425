#!/bin/bash
# compute-sanitizer over the GEMM / attention / model kernels (small shapes)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 17 \
      python tools/sanitize_workload.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize/summary.txt
  tail -5 gpurun_out/sanitize/$tool.log
done

#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_llama.py -q -x > gpurun_out/gemm_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gemm_pytest.log; tail -3 gpurun_out/gemm_pytest.log
ACCO_GEMM_LOG=1 timeout 900 python tools/diag/gemm_model_check.py > gpurun_out/gemm_model.jsonl 2> gpurun_out/gemm_model.err
tail -3 gpurun_out/gemm_model.err
wc -l gpurun_out/gemm_model.jsonl

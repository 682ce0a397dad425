#!/bin/bash
# round 2: 3xTF32 fp32 path — GEMM + model/engine parity tests
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py tests/test_gpu_engine.py tests/test_gpu_llama.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/r2_tf32_pytest.log
cat gpurun_out/r2_tf32_pytest.log

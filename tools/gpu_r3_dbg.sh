#!/bin/bash
cd "$(dirname "$0")/.."
T="tests/test_gpu_model.py::test_wide_row_norm_backward_matches_warp_per_row"
for i in 1 2 3; do timeout 300 python -m pytest -q -m gpu "$T" 2>&1 | tail -1; done
for i in 1 2; do ACCO_GEMM_NO_CG2=1 timeout 300 python -m pytest -q -m gpu "$T" 2>&1 | tail -1; done
ACCO_GEMM_LOG=1 timeout 300 python -m pytest -q -m gpu "$T" -k llama 2>&1 | grep "^gemm" | sort | uniq

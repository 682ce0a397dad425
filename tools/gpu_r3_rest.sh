#!/bin/bash
# the GPU suite from a given test file onwards (after a -x stop)
cd "$(dirname "$0")/.."
timeout 2400 python -m pytest -q -m gpu tests/test_gpu_model.py tests/test_gpu_optim.py tests/test_gpu_peer_multirank.py tests/test_gpu_reference_dropin.py tests/test_gpu_run_api.py tests/test_gpu_lm_acceptance.py > gpurun_out/rest_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/rest_pytest.log; grep -E "passed|failed|FAILED" gpurun_out/rest_pytest.log | tail -5

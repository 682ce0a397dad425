#!/bin/bash
cd "$(dirname "$0")/.."
echo "== old tree"; (cd _old && timeout 600 python -m pytest -q -m gpu tests/test_gpu_model.py -k "attention" 2>&1 | grep -E "passed|failed|FAILED|^E  .*assert" | head -12)
echo "== new tree"; timeout 600 python -m pytest -q -m gpu tests/test_gpu_model.py -k "attention" 2>&1 | grep -E "passed|failed|FAILED|^E  .*assert" | head -12

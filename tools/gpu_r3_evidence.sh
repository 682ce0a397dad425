#!/bin/bash
# End-of-session evidence on the final tree: GPU suite, smoke, bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/r02_gputest_final.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2 | tee -a gpurun_out/r02_gputest_final.txt
bash tools/gpu_r3_final.sh

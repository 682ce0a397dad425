#!/bin/bash
# End-of-session evidence (fourth session): GPU suite + smoke, bench lines, launch list and ncu --set full captures
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_r3_evidence.sh
bash tools/gpu_r3_profile.sh

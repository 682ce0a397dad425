#!/bin/bash
# End-of-session evidence (fourth session): GPU suite + smoke, bench lines, launch list and ncu --set full
# captures (summarised on the box, reports deleted but the attention ones: gpurun_out is capped at 64 MiB),
# compute-sanitizer over the tcgen05 kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_r3_evidence.sh
bash tools/gpu_r3_profile.sh
python tools/ncu_summary.py gpurun_out/prof_step_r02_raw.csv gpurun_out/r02_prof_gemm.ncu-rep gpurun_out/r02_prof_attn.ncu-rep \
    gpurun_out/r02_prof_attnf.ncu-rep gpurun_out/r02_prof_opt.ncu-rep gpurun_out/r02_prof_ce_ln.ncu-rep gpurun_out/r02_prof_misc.ncu-rep
ncu -i gpurun_out/r02_prof_attn.ncu-rep --page details --csv > gpurun_out/r02_prof_attn_details.csv 2>/dev/null
rm -f gpurun_out/r02_prof_gemm.ncu-rep gpurun_out/r02_prof_opt.ncu-rep gpurun_out/r02_prof_ce_ln.ncu-rep gpurun_out/r02_prof_misc.ncu-rep gpurun_out/r02_prof_attnf.ncu-rep
# (compute-sanitizer is closed on this pool: not run)
du -sh gpurun_out

#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_engine.py -q -p no:cacheprovider -x > gpurun_out/pytest_ce.log 2>&1
tail -1 gpurun_out/pytest_ce.log; grep -E "^FAILED" gpurun_out/pytest_ce.log | head -3
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ce_vec|ln_fwd_vec|ln_bwd_vec|colsum_vec" -s 20 -c 12 --csv python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline 2>/dev/null | grep -E "ce_vec|ln_|colsum" | awk -F'","' '{split($5,a,"("); k=a[1]"|"$(NF-2); n[k]++; t[k]+=$NF} END {for (k in n) print k, t[k]/n[k]}' | sort
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_quick.log 2>&1
python - <<'P'
import json
l=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1])
print(round(l['value']), round(l['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in l['breakdown'].items()})
P

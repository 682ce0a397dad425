#!/bin/bash
for v in 8 4 2 1; do
  echo "per_sm $v"
  ACCO_COLSUM_PER_SM=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"colsum_vec" -s 20 -c 12 --csv python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline 2>/dev/null | grep colsum | awk -F'","' '{split($5,a,"("); n[a[1]]++; t[a[1]]+=$NF} END {for (k in n) print "  ", k, t[k]/n[k]/1000, "us"}'
done
for v in 8 2; do
  ACCO_COLSUM_PER_SM=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/b.log 2>&1
  python -c "import json; l=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('per_sm $v', round(l['value']), round(l['ms_per_step'],3))"
done

#!/bin/bash
for v in ACCO_ATTN_SCHED=rr ACCO_ATTN_OVH=1 ACCO_ATTN_OVH=2 ACCO_ATTN_OVH=4; do
  echo "$v"
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_bwd" -s 2 -c 6 --csv python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline 2>/dev/null | grep -E "fa_" | awk -F'","' '{split($5,a,"("); n[a[1]]++; t[a[1]]+=$NF} END {for (k in n) print "  ", k, t[k]/n[k]/1000, "us"}'
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_bwd" -s 2 -c 6 --csv python bench.py --model llama-1b --batch 4 --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline 2>/dev/null | grep -E "fa_" | awk -F'","' '{split($5,a,"("); n[a[1]]++; t[a[1]]+=$NF} END {for (k in n) print "   llama", k, t[k]/n[k]/1000, "us"}'
done

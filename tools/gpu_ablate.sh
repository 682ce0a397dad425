#!/bin/bash
for v in 127 255 128; do
  ACCO_ATTN_ABLATE=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fa_bwd_dkv -s 4 -c 4 --csv python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline 2>/dev/null | grep fa_bwd_dkv | awk -F'","' -v v=$v '{s+=$NF; n++} END {print "ablate", v, s/n, "us"}'
done

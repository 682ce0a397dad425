#!/bin/bash
# epilogue cost: GELU / dGELU GEMMs vs the same shapes with the plain store epilogue
for f in "" "192,1" "256,1"; do
  echo "== force '$f'"
  ACCO_GEMM_FORCE="$f" timeout 120 python tools/gemm_bench.py 768 fc_fwd,fc_fwd_store,fc2_dgrad,fc2_dgrad_store,proj_fwd,head_fwd,head_dgrad,head_wgrad 2>&1 | grep -v total | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(f\"{d['name']:16s} {d['ms']*1000:7.1f}us {d['tflops']:7.1f}\")
    except Exception: pass"
done

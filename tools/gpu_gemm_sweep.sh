#!/bin/bash
# per-shape tile sweep of the tcgen05 GEMM (GPT-2 small shapes)
for f in "" "128,1" "192,1" "256,1"; do
  echo "== force '$f'"
  ACCO_GEMM_FORCE="$f" timeout 120 python tools/gemm_bench.py 768 qkv_fwd,proj_fwd,fc_fwd,fc2_fwd,fc2_dgrad,fc_dgrad,qkv_dgrad 2>&1 | grep -v total | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(f\"{d['name']:12s} {d['ms']*1000:7.1f}us {d['tflops']:7.1f}\")
    except Exception: pass"
done
for f in "" "128,1" "128,2" "128,4" "192,2" "192,4" "256,2" "256,4" "128,8"; do
  echo "== force '$f'"
  ACCO_GEMM_FORCE="$f" timeout 120 python tools/gemm_bench.py 768 proj_wgrad,qkv_wgrad,fc_wgrad,fc2_wgrad 2>&1 | grep -v total | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(f\"{d['name']:12s} {d['ms']*1000:7.1f}us {d['tflops']:7.1f}\")
    except Exception: pass"
done

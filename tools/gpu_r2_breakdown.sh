#!/bin/bash
# per-class step breakdown with / without the emulated 8-GPU comm (CLC on)
cd "$(dirname "$0")/.."
for emu in "" "--emulate-comm-gpus 8 --emulate-ctas 16"; do
  python bench.py --steps 15 --warmup 4 --no-cpu-baseline --no-baselines $emu 2>&1 | tail -1 | \
  python -c "import sys,json; l=json.loads(sys.stdin.read()); print('$emu', round(l['value']), round(l['ms_per_step'],2), {k: round(v['ms_per_step'],3) for k,v in l['breakdown'].items()})"
done

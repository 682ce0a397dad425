#!/bin/bash
timeout 300 python tools/gemm_bench.py 768 > gpurun_out/gemm_bench_768.log 2>&1; cat gpurun_out/gemm_bench_768.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_a.log 2>&1
ACCO_SERIAL_REDUCE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_serial.log 2>&1
for f in bench_a bench_serial; do python - $f <<'P'
import json,sys
l=json.loads(open(f'gpurun_out/{sys.argv[1]}.log').read().strip().splitlines()[-1])
print(sys.argv[1], round(l['value']), round(l['ms_per_step'],3), 'gemm frac', round(l['roofline']['frac'],3), {k:round(v['ms_per_step'],3) for k,v in l['breakdown'].items()})
P
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fa_|dsum" -s 20 -c 4 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 1 --profile --no-baselines --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1
tail -3 gpurun_out/ncu_attn.log

timeout 900 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1
grep -E "passed|failed|FAILED|Error |error:" gpurun_out/pytest_quick.log | head -30
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_quick.log 2>&1
python - <<'P'
import json
l=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1])
print(l['value'], l['ms_per_step'], l['roofline']['frac'], json.dumps(l['attention']), json.dumps(l['roofline_optimizer'])[:200])
for k,v in l.get('breakdown',{}).items(): print(k, round(v['ms_per_step'],3), round(v['share_of_step'],3))
P

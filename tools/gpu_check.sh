timeout 300 python -m pytest tests/test_gpu_model.py tests/test_gpu_engine.py tests/test_gpu_comm.py tests/test_gpu_gemm.py -q -p no:cacheprovider -x > gpurun_out/pytest_quick.log 2>&1
grep -E "passed|failed|FAILED|Error |error:" gpurun_out/pytest_quick.log | head -30
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/bench_quick.log 2>&1
python - <<'P'
import json
l=json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1])
print(l['value'], l['ms_per_step'], l['roofline']['frac'], json.dumps(l['attention']))
for k,v in l.get('breakdown',{}).items(): print(k, round(v['ms_per_step'],3), round(v['share_of_step'],3))
P
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-baselines --profile > /dev/null 2>&1
python - <<'P'
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_q.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[hi+1:]:
    try: agg[r[ki].split('(')[0].replace('void ','').replace('unnamed>::','')].append(float(r[vi].replace(',','')))
    except Exception: pass
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])): print(f"{k[:40]:40s} {len(v):5d} {sum(v)/len(v)/1e3:8.2f} us avg {sum(v)/1e3:9.1f} us tot")
P

ls gpurun_out/

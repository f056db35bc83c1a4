# gpurun helper: quick tests, bench, and a per-kernel launch list (ncu durations)
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "${PYTEST_K:-score or step}" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_bd.json 2>gpurun_out/bench_bd.err; python -c "
import json; d=json.load(open('gpurun_out/bench_bd.json')); print('step_us', round(d['value'],1), 'calls', {k: round(v*1000,1) for k,v in d['per_call_ms'].items()}, 'roof', round(d['roofline']['frac'],3))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bd.csv python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_bd.csv')) if len(r)>5]
h={k:i for i,k in enumerate(rows[0])}
agg={}
for r in rows[1:]:
    n=r[h['Kernel Name']]
    if any(x in n for x in ('elementwise','kv_kernel','query_kernel','Fill')): continue
    k=n.split('(')[0].split('::')[-1][:28]
    agg.setdefault(k,[]).append(float(r[h['Metric Value']])/1000)
for k,v in agg.items(): print(f'{k:30s} n={len(v)} mean_us={sum(v)/len(v):8.1f}')
PY

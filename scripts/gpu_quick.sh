# quick GPU iteration: a test subset (PYTEST_K), select phase profile, short bench lines
TAG=${TAG:-q}
if [ -n "$PYTEST_K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "$PYTEST_K" > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${TAG}_pytest.txt
fi
[ -n "$PROF_SELECT" ] && timeout 300 python scripts/prof_select.py 2>&1 | tail -22
for P in ${SHARDS:-1 8}; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-a5 --steps 20 --emulate-shard $P > gpurun_out/${TAG}_bench_p$P.json 2>gpurun_out/${TAG}_bench_p$P.err
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench_p$P.json'))
print('P=$P', 'us/step %.1f' % d['value'], 'per_call_us', {k: round(v*1e3,1) for k,v in d['per_call_ms'].items()}, 'p10/50/90', [round(x,1) for x in d['step_us_p10_p50_p90']])" || tail -5 gpurun_out/${TAG}_bench_p$P.err
done

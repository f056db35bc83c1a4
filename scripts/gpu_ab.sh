# A/B timing: eager 20-step (round-1 method) vs graph-replay headline, P = 1 and 8
TAG=${TAG:-ab}
for P in 1 8; do
  for MODE in "--eager --steps 20 --warmup 5" "--steps 300 --warmup 10"; do
    timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-a5 --emulate-shard $P $MODE > gpurun_out/${TAG}.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/${TAG}.json'))
print('P=$P', '$MODE'.split()[0], 'us/step %.1f' % d['value'], {k: round(v*1e3,1) for k,v in d['per_call_ms'].items()}, d['clocks'].get('reasons'))"
  done
done

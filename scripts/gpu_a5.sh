# a5 schedules: stream priority none / main / side, with and without the forward, P = 1 and 8
for P in 1 8; do for PR in none main side; do for F in "" "--a5-no-forward"; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --emulate-shard $P --a5-priority $PR $F > gpurun_out/a5x.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/a5x.json').read().strip().splitlines()[-1]); a=d['a5']
print('P=$P prio=$PR fwd=${F:-yes}', 'serial %.1f pipelined %.1f gain %.3f' % (a['serial_us'], a['pipelined_us'], a['pipelined_gain_frac']))"
done; done; done

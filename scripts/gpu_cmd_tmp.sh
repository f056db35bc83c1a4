for P in 1 8; do for L in paper_2510_07486_b200/libasyncspade.so build/ab/lag3/libasyncspade.so build/ab/lag4/libasyncspade.so; do
ASYNCSPADE_LIB=$PWD/$L timeout 120 python bench.py --no-cpu-baseline --no-e2e --no-a5 --steps 20 --emulate-shard $P 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$L P=$P', 'us/step %.1f' % d['value'], {k: round(v*1e3,1) for k,v in d['per_call_ms'].items()})"
done; done
for L in build/ab/lag3/libasyncspade.so build/ab/lag4/libasyncspade.so; do
ASYNCSPADE_LIB=$PWD/$L timeout 300 python scripts/sweep.py high-concurrency --only 512 --out gpurun_out/t_hc.jsonl > /dev/null 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/t_hc.jsonl').readline()); print('$L b512', round(d['us_per_step'],1), 't_dec', round(d['t_dec'],1))"
done
ASYNCSPADE_LIB=$PWD/build/ab/lag4/libasyncspade.so timeout 600 python -m pytest tests -m gpu -q -x -k "decode or step_qwen3 or high or group" 2>&1 | tail -1

# session-3 quick experiments: paged bench lines (PAGES), select phase profile (PROF_SELECT=1)
TAG=${TAG:-s3}
if [ -n "$PYTEST_K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "$PYTEST_K" > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${TAG}_pytest.txt
fi
for PG in $PAGES; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-a5 --steps 20 --paged $PG > gpurun_out/${TAG}_paged$PG.json 2>gpurun_out/${TAG}_paged$PG.err
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}_paged$PG.json'))
print('page $PG', 'us/step %.1f' % d['value'], {k: round(v*1e3,1) for k,v in d['per_call_ms'].items()})" || tail -5 gpurun_out/${TAG}_paged$PG.err
done
[ -n "$PROF_SELECT" ] && timeout 300 python scripts/prof_select.py 2>&1 | tail -30
[ -n "$EXTRA" ] && eval "$EXTRA"
true

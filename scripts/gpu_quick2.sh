timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "${PYTEST_K:-predict or step}" > gpurun_out/pytest_quick.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_quick.txt
for P in ${SHARDS:-1 8}; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --emulate-shard $P > gpurun_out/shard$P.json 2>gpurun_out/shard$P.err; echo "P=$P rc=$?"; tail -2 gpurun_out/shard$P.err
  python -c "import json;d=json.load(open('gpurun_out/shard$P.json'));print($P, round(d['value'],1), d['per_call_ms'], round(d['roofline_frac_step'],3))"
done
if [ -n "$LAUNCHES" ]; then for P in $LAUNCHES; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p$P.csv python bench.py --profile --steps 2 --warmup 1 --emulate-shard $P > /dev/null 2>&1; grep -v -E "elementwise|FillFunctor|kv_kernel|query_kernel" gpurun_out/launches_p$P.csv | tail -5 | awk -F'","' '{print $5, $NF}' | cut -c1-50,150-; done; fi

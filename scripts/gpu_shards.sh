# Per-GPU work of the P-way KV-head split (emulated on one GPU) + predict phase profile
for P in 1 2 4 8; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --emulate-shard $P > gpurun_out/shard$P.json 2>gpurun_out/shard$P.err; echo "P=$P rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/shard$P.json'));print($P, round(d['value'],1), d['per_call_ms'], round(d['roofline_frac_step'],3))"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p8.csv python bench.py --profile --steps 2 --warmup 1 --emulate-shard 8 > /dev/null 2>&1
grep -v -E "elementwise|FillFunctor" gpurun_out/launches_p8.csv | tail -5 | awk -F'","' '{print $5, $NF}'
timeout 120 python scripts/exp_predict_prof.py

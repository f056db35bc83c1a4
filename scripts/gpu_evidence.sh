# One gpurun call for the round's evidence: GPU tests, smoke(), a full bench
# line (cpu_baseline, e2e, a5), the reference arm, the ncu launch list, one
# ncu --set full capture of each of the step's kernels (second step, warm),
# emulated P-way shards, ragged and paged bench lines.  Summaries are made
# locally (scripts/make_profiles.py).
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method thread > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.txt
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1; echo "reference rc=$?"; cut -c1-300 gpurun_out/${TAG}_bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"predict|score_tc|select_kernel|decode_tc|decode_combine" -s 5 -c 5 -o gpurun_out/${TAG}_full python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/${TAG}_ncu_full.log
rm -f gpurun_out/${TAG}_scaling_emulated.jsonl
for P in 2 4 8; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --emulate-shard $P >> gpurun_out/${TAG}_scaling_emulated.jsonl 2>/dev/null; done; echo "shards done"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_p8.csv python bench.py --profile --steps 2 --warmup 1 --emulate-shard 8 > /dev/null 2>&1; echo "launches p8 rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-a5 --ragged > gpurun_out/${TAG}_bench_ragged.json 2>/dev/null; echo "ragged rc=$?"
rm -f gpurun_out/${TAG}_bench_paged.jsonl
for P in 16 32 64 128; do timeout 300 python bench.py --no-cpu-baseline --paged $P >> gpurun_out/${TAG}_bench_paged.jsonl 2>/dev/null; done; echo "paged done"
timeout 300 python scripts/sweep.py gather --out gpurun_out/${TAG}_sweep_gather.jsonl > /dev/null 2>&1; echo "gather sweep rc=$?"

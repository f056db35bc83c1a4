# One gpurun call for the round's evidence: GPU tests, a full bench line (with
# cpu_baseline and e2e), the ncu launch list and one ncu --set full capture of
# each of the step's kernels (second step, warm).  Summaries are made locally.
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.txt
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"predict|score_tc|select_kernel|decode_tc|decode_combine" -s 5 -c 5 -o gpurun_out/${TAG}_full python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/${TAG}_ncu_full.log
# per-GPU work of the P-way KV-head split, emulated on this one GPU (scaling evidence)
for P in 2 4 8; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --emulate-shard $P >> gpurun_out/${TAG}_scaling_emulated.jsonl 2>/dev/null; done; echo "shards done"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_p8.csv python bench.py --profile --steps 2 --warmup 1 --emulate-shard 8 > /dev/null 2>&1; echo "launches p8 rc=$?"

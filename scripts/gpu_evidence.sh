# One gpurun call for a round's evidence: GPU tests, smoke(), the bench line
# (cpu_baseline on all host cores, e2e, a5 with the layer forward, sustained),
# the reference arm, the ncu launch list, one ncu --set full capture of each
# of the step's kernels (warm second step), an L2-residency pass
# (--cache-control none), emulated P-way shards, ragged and paged lines.
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
[ -z "$SKIP_TESTS" ] && { timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.txt; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cut -c1-400 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1; echo "reference rc=$?"; cut -c1-300 gpurun_out/${TAG}_bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --profile --eager --steps 2 --warmup 1 --no-a5 > /dev/null 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"predict|score_tc|select_kernel|decode_tc|decode_combine" -s 5 -c 5 -o gpurun_out/${TAG}_full python bench.py --profile --eager --steps 2 --warmup 1 --no-a5 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/${TAG}_ncu_full.log
timeout 900 ncu --replay-mode application --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum \
  -k regex:"score_tc|select_kernel|decode_tc|decode_combine|predict" -s 10 -c 10 --csv --log-file gpurun_out/${TAG}_l2.csv \
  python bench.py --profile --eager --steps 3 --warmup 2 --no-a5 > gpurun_out/${TAG}_l2.log 2>&1; echo "ncu l2 rc=$?"
rm -f gpurun_out/${TAG}_scaling_emulated.jsonl
for P in 2 4 8; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --emulate-shard $P >> gpurun_out/${TAG}_scaling_emulated.jsonl 2>/dev/null; done; echo "shards done"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_p8.csv python bench.py --profile --eager --steps 2 --warmup 1 --emulate-shard 8 --no-a5 > /dev/null 2>&1; echo "launches p8 rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-a5 --ragged > gpurun_out/${TAG}_bench_ragged.json 2>/dev/null; echo "ragged rc=$?"
rm -f gpurun_out/${TAG}_bench_paged.jsonl
for P in 16 32 64 128; do timeout 300 python bench.py --no-cpu-baseline --paged $P >> gpurun_out/${TAG}_bench_paged.jsonl 2>/dev/null; done; echo "paged done"
for C in qwen3-8b_b32_ctx32k mla16_b16_ctx32k mqa64_b32_ctx32k; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-a5 --config $C >> gpurun_out/${TAG}_bench_variants.jsonl 2>/dev/null; done; echo "variants done"

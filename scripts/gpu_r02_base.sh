# Round-2 baseline: GPU tests, one bench line, and an L2-residency ncu pass
# (application replay, --cache-control none, so the score buffer's L2 state
# between score and select is the live one).
TAG=${TAG:-r02a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" ; python -c "import os;print('affinity', len(os.sched_getaffinity(0)))"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json | cut -c1-1500
timeout 900 ncu --replay-mode application --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum \
  -k regex:"score_tc|select_kernel|decode_tc|decode_combine|predict" -s 10 -c 10 --csv --log-file gpurun_out/${TAG}_l2.csv \
  python bench.py --profile --steps 3 --warmup 2 > gpurun_out/${TAG}_l2.log 2>&1; echo "ncu l2 rc=$?"; tail -3 gpurun_out/${TAG}_l2.log

# gpurun helper: selected GPU tests (PYTEST_K) with a hard timeout, then optional bench
timeout ${T:-300} python -m pytest tests/test_gpu_parity.py -q -x -rf -k "${PYTEST_K:-score}" > gpurun_out/pytest_quick.txt 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_quick.txt
if [ -n "$BENCH" ]; then timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err; echo "bench rc=$?"; cat gpurun_out/bench_quick.json; tail -3 gpurun_out/bench_quick.err; fi

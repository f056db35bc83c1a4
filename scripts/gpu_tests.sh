# gpurun helper: GPU test suite only, full report in gpurun_out/pytest_gpu_full.txt
timeout 1200 python -m pytest tests -m gpu -q -rf ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu_full.txt 2>&1
tail -15 gpurun_out/pytest_gpu_full.txt

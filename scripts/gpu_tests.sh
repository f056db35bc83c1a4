# GPU test suite (optionally a subset: PYTEST_ARGS), full report under gpurun_out/
TAG=${TAG:-r02}
timeout ${T:-1500} python -m pytest tests -m gpu -q -rf --timeout 600 ${PYTEST_ARGS:-} > gpurun_out/${TAG}_pytest.txt 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/${TAG}_pytest.txt

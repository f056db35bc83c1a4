# GPU test suite, or a subset: PYTEST_ARGS='tests/x.py -k "a or b"' (eval'd, so quote -k); report under gpurun_out/
TAG=${TAG:-r02}
eval timeout ${T:-1500} python -m pytest ${PYTEST_ARGS:-tests} -m gpu -q -rf --timeout 600 > gpurun_out/${TAG}_pytest.txt 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/${TAG}_pytest.txt

# Session-3 baseline: full GPU suite, smoke, P=1 / P=8 bench lines
TAG=${TAG:-s3a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/${TAG}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash scripts/gpu_quick.sh

timeout 900 python -m pytest tests -m gpu -q -x -k "select or long or step or quest or high" > gpurun_out/t_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_pytest.txt
SHARDS=1,8 timeout 300 python scripts/prof_select.py 2>&1 | grep -E "P=|radix|alone|fallback"
CONFIG=long-cot_b8_ctx524288 SHARDS=8 timeout 300 python scripts/prof_select.py 2>&1 | grep -E "P=|radix|alone|fallback"
bash scripts/gpu_quick.sh
timeout 600 python scripts/sweep.py long-cot --only 19 --out gpurun_out/t_lc.jsonl > /dev/null 2>&1; cut -c1-200 gpurun_out/t_lc.jsonl
timeout 300 python scripts/sanitize_small.py 2>&1 | tail -5
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_small.py 2>&1 | tail -5

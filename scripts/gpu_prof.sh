# gpurun helper: full GPU tests + launch list + ncu --set full of named kernels
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_full.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1
grep -v -E "elementwise|FillFunctor|kv_kernel|query_kernel" gpurun_out/launches.csv | awk -F'","' '{print $5, $NF}' | cut -c1-60,200- | tail -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-score_tc|select_kernel|decode_partial|predict_kernel}" -s 4 -c 4 -o gpurun_out/prof python bench.py --profile --steps 2 --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log

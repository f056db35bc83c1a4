# gpurun helper: ncu --set full of kernels matching KREGEX during a short bench run
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-2} -o gpurun_out/${OUT:-prof} python bench.py --profile --steps 1 --warmup 1 ${BENCH_ARGS:-} > gpurun_out/ncu_${OUT:-prof}.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${OUT:-prof}.log

# ncu --set full of one kernel family AS IT RUNS in the step (--cache-control
# none: L2 keeps the previous kernel's output, e.g. the score buffer select
# reads), source-level, at config [2] P = 1 and the P = 8 shard.
TAG=${TAG:-live}
K=${KREGEX:-select_kernel}
for P in ${SHARDS:-1 8}; do
  timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:"$K" -s ${SKIP:-3} -c ${COUNT:-1} \
    -o gpurun_out/${TAG}_p${P} python bench.py --profile --eager --steps 2 --warmup 1 --emulate-shard $P --no-a5 > gpurun_out/${TAG}_p${P}.log 2>&1
  echo "ncu P=$P rc=$?"; tail -1 gpurun_out/${TAG}_p${P}.log
done

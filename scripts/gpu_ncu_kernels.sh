# ncu --set full captures (source-level) of the step's latency-bound kernels:
# select / predict / decode / combine at config [2] P = 1 and the P = 8 shard.
TAG=${TAG:-r02c}
K=${KREGEX:-"predict|select_kernel|decode_tc|decode_combine"}
for P in ${SHARDS:-1 8}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -s ${SKIP:-4} -c ${COUNT:-4} \
    -o gpurun_out/${TAG}_p${P} python bench.py --profile --steps 2 --warmup 1 --emulate-shard $P --no-a5 > gpurun_out/${TAG}_p${P}.log 2>&1
  echo "ncu P=$P rc=$?"; tail -2 gpurun_out/${TAG}_p${P}.log
done

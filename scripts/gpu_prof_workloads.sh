# launch lists (ncu, one eager step) of the wider workloads: high concurrency
# b512 / b1, long-CoT 512k shard, paged P=16, MLA / MQA variants
TAG=${TAG:-wl}
run() { name=$1; shift
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_${name}.csv \
    python bench.py --profile --eager --steps 2 --warmup 1 --no-a5 "$@" > /dev/null 2>&1; echo "$name rc=$?"; }
run hc512 --config high-conc_b512_ctx4k
run hc1 --config high-conc_b1_ctx4k
run lc512k --config long-cot_b8_ctx524288 --emulate-shard 8
run paged16 --paged 16
run mla16 --config mla16_b16_ctx32k
run mqa64 --config mqa64_b32_ctx32k

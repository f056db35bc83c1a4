# the round's sweeps (configs [3], [4], NEXT-1/2/4, group sizes) -> gpurun_out/${TAG}_sweep_*.jsonl
TAG=${TAG:-r02}
for S in ${SWEEPS:-long-cot high-concurrency layer-packed groups gather quest}; do
  timeout 900 python scripts/sweep.py $S --out gpurun_out/${TAG}_sweep_${S}.jsonl > /dev/null 2> gpurun_out/${TAG}_sweep_${S}.err
  echo "sweep $S rc=$?"
done

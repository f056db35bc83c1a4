# gpurun helper: per-kernel durations (ncu, duration only) of one bench step
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python bench.py --profile --steps 1 --warmup 1 ${BENCH_ARGS:-} > /dev/null 2>&1
python - <<'PY'
import csv
lines = open("gpurun_out/launches_q.csv").read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
keep = [r for r in rows[1:] if any(k in r[h.index("Kernel Name")] for k in ("predict_kernel", "score_tc", "select_kernel", "decode_tc", "decode_combine"))]
for r in keep[-5:]:
    print(f'{r[h.index("Kernel Name")][:50]:50s} {float(r[h.index("Metric Value")].replace(",", ""))/1e3:8.1f} us')
PY

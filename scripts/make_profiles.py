"""Turn a round's gpurun_out/ evidence into the committed profiles/ summaries.
usage: python scripts/make_profiles.py r01"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")
rep = os.path.join(src, f"{tag}_full.ncu-rep")

# 1. per-kernel dram traffic from the --set full capture
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}
per = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    short = name.split("::")[1].split("(")[0].split("<")[0] if "::" in name else name
    val = lambda m: float(r[h.index(m)]) * scale[units[h.index(m)]]
    per[short] = {"dram_read": val("dram__bytes_read.sum"), "dram_write": val("dram__bytes_write.sum"),
                  "duration_s": val("gpu__time_duration.sum")}
traffic = {"source": f"profiles/{tag}_ncu_summary.txt (ncu --set full, one launch each, second step)",
           "per_kernel": per,
           "score_select_dram_bytes_per_launch":
               sum(per[k]["dram_read"] + per[k]["dram_write"] for k in ("score_tc_kernel", "select_kernel"))}
with open(os.path.join(dst, "ncu_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1)

# 2. summary text: key metrics per kernel
summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                      capture_output=True, text=True).stdout
with open(os.path.join(dst, f"{tag}_ncu_summary.txt"), "w") as f:
    f.write(f"# ncu --set full --clock-control none, bench.py --profile (config [2]), {tag}\n")
    f.write("# kernel: dram read / write bytes per launch, duration\n")
    for k, v in per.items():
        f.write(f"#   {k:24s} read {v['dram_read']/1e6:10.2f} MB  write {v['dram_write']/1e6:8.2f} MB"
                f"  {v['duration_s']*1e6:8.2f} us\n")
    f.write(summ)

# 3. launch list (ours only) with each kernel's share of the step
lines = open(os.path.join(src, f"{tag}_launches.csv")).read().splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
keep = [r for r in rows[1:] if any(k in r[h.index("Kernel Name")] for k in
        ("predict_", "score_tc", "select_kernel", "decode_tc", "decode_combine"))]
with open(os.path.join(dst, f"{tag}_launches.csv"), "w") as f:
    w = csv.writer(f)
    w.writerow(["ID", "Kernel Name", "gpu__time_duration.sum (ns)"])
    for r in keep:
        w.writerow([r[h.index("ID")], r[h.index("Kernel Name")][:90], r[h.index("Metric Value")]])
    last = keep[-5:]            # predict, score, select, decode, combine of the last step
    tot = sum(float(r[h.index("Metric Value")].replace(",", "")) for r in last)
    f.write("# share of the last step (serialised, cold-cache ncu times):\n")
    for r in last:
        v = float(r[h.index("Metric Value")].replace(",", ""))
        f.write(f"# {r[h.index('Kernel Name')][:40]}: {v/1e3:.1f} us = {100*v/tot:.1f}%\n")
print(json.dumps(traffic, indent=1))


# 4. L2 residency (application replay, --cache-control none)
l2 = os.path.join(src, f"{tag}_l2.csv")
if os.path.exists(l2):
    import collections
    rows = list(csv.reader(open(l2)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    d = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d.setdefault((int(r[h.index("ID")]), r[h.index("Kernel Name")].split("(")[0].replace("void <unnamed>::", "")),
                     {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    with open(os.path.join(dst, f"{tag}_l2_residency.txt"), "w") as f:
        f.write("# L2 residency of the score buffer and the decode partials (SURVEY §8(d)), config [2]:\n")
        f.write("# ncu --replay-mode application --cache-control none --clock-control none (the step's\n")
        f.write("# kernels as they run back to back: nothing flushes L2 between producer and consumer).\n")
        f.write("%-4s %-26s %9s %12s %12s %10s %10s %7s\n" % ("id", "kernel", "dur_us", "dram_rd_MB",
                                                          "dram_wr_MB", "L2rd_MB", "L2hit_MB", "hit%"))
        for (i, k), m in d.items():
            rd = m["lts__t_sectors_srcunit_tex_op_read.sum"] * 32 / 1e6
            hit = m["lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum"] * 32 / 1e6
            f.write("%-4d %-26s %9.1f %12.2f %12.2f %10.1f %10.1f %7.1f\n" % (
                i, k[:26], m["gpu__time_duration.sum"] / 1e3, m["dram__bytes_read.sum"] / 1e6,
                m["dram__bytes_write.sum"] / 1e6, rd, hit, 100 * hit / max(rd, 1e-9)))
        f.write("# 'lookup miss' sectors that do not reach DRAM are served by the far L2 partition\n")

# 5. the bench lines
import shutil
for name in ("bench.json", "bench_reference.json", "bench_ragged.json", "scaling_emulated.jsonl",
             "bench_paged.jsonl", "bench_variants.jsonl", "launches_p8.csv"):
    p_src = os.path.join(src, f"{tag}_{name}")
    if os.path.exists(p_src):
        shutil.copy(p_src, os.path.join(dst, f"{tag}_{name}"))

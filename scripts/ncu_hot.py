"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.
usage: python scripts/ncu_hot.py report.ncu-rep kernel-regex [N]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(lines[1:]))
h = {k: i for i, k in enumerate(rows[0])}
data = []
for r in rows[1:]:
    try:
        data.append((int(r[h["Warp Stall Sampling (All Samples)"]]), r[h["Address"]][-5:],
                     r[h["Source"]].strip()[:90]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for s, a, src in sorted(data, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}%  {a}  {src}")

"""Summarise an ncu report: per kernel, key SOL / occupancy / stall metrics.
usage: python scripts/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = {k: i for i, k in enumerate(rows[0])}
KEEP = re.compile(r"Duration|Memory Throughput|DRAM Throughput|Compute \(SM\) Throughput|"
                  r"Achieved Occupancy|Theoretical Occupancy|Registers Per Thread|"
                  r"Issue Slots Busy|Eligible Warps|Warp Cycles Per Issued|No Eligible|"
                  r"L2 Hit Rate|L1/TEX Hit|Dynamic Shared|Block Limit|Executed Ipc A")
seen = {}
for r in rows[1:]:
    if len(r) < 15:
        continue
    kid = (r[h["ID"]], r[h["Kernel Name"]][:60])
    if pat and not pat.search(kid[1]):
        continue
    if KEEP.search(r[h["Metric Name"]]):
        seen.setdefault(kid, []).append(f'{r[h["Metric Name"]]}={r[h["Metric Value"]]}{r[h["Metric Unit"]]}')
    if r[h["Rule Name"]] and r[h["Rule Type"]] in ("OPT", "WRN") and "Stall" in r[h["Rule Description"]][:400]:
        seen.setdefault(kid, []).append("RULE: " + r[h["Rule Description"]][:300])
for k, v in seen.items():
    print("==", k[0], k[1])
    for x in v:
        print("   ", x)

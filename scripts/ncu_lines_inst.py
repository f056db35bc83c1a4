"""Per-source-line executed warp instructions (ncu source page), top N.
usage: python scripts/ncu_lines_inst.py report kernel-regex [N]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
agg, fname, cur, hdr = {}, "?", None, None
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = {k: i for i, k in enumerate(r)}; continue
    if hdr is None: continue
    try: s = int(r[hdr["Instructions Executed"]])
    except (ValueError, IndexError, KeyError): s = 0
    if r[0].strip(): cur = (fname, r[0], r[1].strip()[:80])
    if cur: agg[cur] = agg.get(cur, 0) + s
tot = sum(agg.values()) or 1
print(f"total warp instructions: {tot}")
for (f, ln, src), s in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{100 * s / tot:5.1f}%  {f}:{ln}  {src}")

"""Per-kernel SASS counts that prove the tensor-core / TMA / async paths.
usage: python scripts/sass_evidence.py > profiles/r01_sass_evidence.txt"""
import os, re, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2510_07486_b200", "libasyncspade.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "LDGSTS", "DMMA", "SYNCS", "ELECT", "ATOMS", "MUFU.EX2"]
print("# SASS evidence (cuobjdump -sass paper_2510_07486_b200/libasyncspade.so), sm_100a")
print("# per kernel: counts of the instructions that prove the tensor-core / TMA / async paths")
print("# UTCHMMA = tcgen05.mma (kind::f16), UTCBAR = tcgen05.commit, LDTM = tcgen05.ld,")
print("# UTMALDG = TMA tensor load, UBLKCP = cp.async.bulk, LDGSTS = cp.async, DMMA = fp64 mma.sync,")
print("# SYNCS = mbarrier ops, ELECT = elect.sync, ATOMS = shared atomics")
for block in re.split(r"\n\s*Function : ", out)[1:]:
    name = block.split("\n", 1)[0].strip()
    counts = {op: len(re.findall(r"\b" + re.escape(op) + r"(?:\.|\s)", block)) for op in OPS}
    s = "  ".join(f"{k}={v}" for k, v in counts.items() if v)
    if s:
        print(name, s)

"""Bisect predict fast-path non-finite inputs (each case in its own process)."""
import subprocess, sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys, numpy as np, torch
nan = float("nan"); inf = float("inf")
sys.path.insert(0, "%s")
import paper_2510_07486_b200 as asp
B, H, W, D, r, val, flags = %r
bad = np.ones((B, H, W, 64 if D == 64 else D), np.float32)
bad += np.random.default_rng(0).standard_normal(bad.shape).astype(np.float32) * 0.1
if r >= 0: bad[0, r, 2, 5] = val
fl = torch.zeros(1, dtype=torch.int32, device="cuda")
g = asp.predict_query(torch.from_numpy(bad).cuda(), dev_flags=fl, flags=flags).cpu().numpy()
print("ok flags", fl.item(), np.isfinite(g).all(axis=-1).tolist())
'''
cases = [(1, 2, 4, 64, 1, float("nan"), 0), (1, 2, 4, 64, 0, float("nan"), 0), (1, 2, 4, 64, -1, 0.0, 0),
         (1, 2, 4, 64, 1, float("inf"), 0), (1, 2, 16, 128, 1, float("nan"), 0),
         (1, 2, 4, 64, 1, float("nan"), 1), (1, 1, 4, 64, 0, float("nan"), 0)]
for c in cases:
    try:
        r = subprocess.run([sys.executable, "-c", CASE % (ROOT, c)], capture_output=True, text=True, timeout=60)
        print(c, r.stdout.strip()[-200:], r.stderr.strip()[-300:])
    except subprocess.TimeoutExpired:
        print(c, "HANG")

"""Predict fast path with a non-finite window in one row of a pair: flags and
per-row outputs vs the oracle / passthrough."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_07486_b200 as asp, oracle
for flags in (asp.ASSEMBLY_SINGLE, 0):
    for r in (1, 0):
        bad = np.ones((1, 2, 4, 64), np.float32) + np.random.default_rng(0).standard_normal((1, 2, 4, 64)).astype(np.float32) * 0.1
        bad[0, r, 2, 5] = np.nan
        fl = torch.zeros(1, dtype=torch.int32, device="cuda")
        g = asp.predict_query(torch.from_numpy(bad).cuda(), dev_flags=fl, flags=flags).cpu().numpy()
        ref, cond = oracle.predict(bad, 1e-2, flags, 0)
        print("flags", flags, "nan row", r, "dev_flags", fl.item(), "oracle cond", cond,
              [float(np.abs(g[0, i] - ref[0, i]).max()) for i in range(2)],
              [bool(np.array_equal(g[0, i], bad[0, i, 3])) for i in range(2)], flush=True)

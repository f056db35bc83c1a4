import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["ASYNCSPADE_LIB"] = os.path.join(ROOT, "build/prof/libasyncspade_prof.so")
import paper_2510_07486_b200 as asp
bad = np.ones((1, 2, 4, 64), np.float32) + np.random.default_rng(0).standard_normal((1, 2, 4, 64)).astype(np.float32) * 0.1
bad[0, 0, 2, 5] = np.nan
fl = torch.zeros(1, dtype=torch.int32, device="cuda")
g = asp.predict_query(torch.from_numpy(bad).cuda(), dev_flags=fl, flags=asp.ASSEMBLY_SINGLE).cpu().numpy()
torch.cuda.synchronize()
print("dev_flags", fl.item())

"""Each call of the config [2] step timed in isolation (K back-to-back calls
of the same entry point) vs the whole step."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
cfg = configs.QWEN3_32B
s = DecodeStep(cfg, "cuda")
s.fill_synthetic()
s.run()
K = 20
def timeit(f):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3
pred = lambda: asp.predict_query(s.window, s.q_hat, dev_flags=s.dev_flags, params=s.p_pred)
sel = lambda: asp.score_select(s.q_hat, s.k_cache, s.seq_lens, cfg.top_k, sel_idx=s.sel_idx,
                               workspace=s.ws_sel, dev_flags=s.dev_flags, params=s.p_sel)
dec = lambda: asp.sparse_decode(s.q, s.k_cache, s.v_cache, s.seq_lens, s.sel_idx, out=s.out,
                                workspace=s.ws_dec, params=s.p_dec)
for name, f in [("predict", pred), ("score_select", sel), ("decode", dec), ("step", s.run)]:
    print(f"{name:14s} {timeit(f):8.1f} us")

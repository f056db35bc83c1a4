"""score_select back to back vs with an L2 flush in between (config [2])."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
cfg = configs.QWEN3_32B
step = DecodeStep(cfg, "cuda")
step.fill_synthetic()
asp.predict_query(step.window, step.q_hat, params=step.p_pred)
f = lambda: asp.score_select(step.q_hat, step.k_cache, step.seq_lens, cfg.top_k, sel_idx=step.sel_idx,
                             workspace=step.ws_sel, params=step.p_sel)
junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3): f()
for mode in ("back-to-back", "flush-between"):
    ts = []
    for i in range(8):
        if mode == "flush-between":
            junk.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(mode, " ".join(f"{t:.0f}" for t in ts))

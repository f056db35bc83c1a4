"""select time vs cluster size (instrumented build honours ASP_SELECT_CLUSTER)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ASYNCSPADE_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build/prof/libasyncspade_prof.so")
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
cfg = configs.by_name(sys.argv[1])
step = DecodeStep(cfg, "cuda")
step.fill_synthetic()
asp.predict_query(step.window, step.q_hat, params=step.p_pred)
f = lambda: asp.score_select(step.q_hat, step.k_cache, step.seq_lens, cfg.top_k, sel_idx=step.sel_idx,
                             workspace=step.ws_sel, params=step.p_sel)
for _ in range(3): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): f()
e1.record(); torch.cuda.synchronize()
print(cfg.name, os.environ.get("ASP_SELECT_CLUSTER"), f"{e0.elapsed_time(e1) / 10 * 1e3:.1f} us")

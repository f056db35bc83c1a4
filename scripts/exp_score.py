"""Time asyncspade_score_select alone (config [2]) under the current env."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
step = DecodeStep(configs.QWEN3_32B, "cuda")
step.fill_synthetic()
asp.predict_query(step.window, step.q_hat, params=step.p_pred)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    asp.score_select(step.q_hat, step.k_cache, step.seq_lens, 2048, sel_idx=step.sel_idx, workspace=step.ws_sel, params=step.p_sel)
torch.cuda.synchronize()
ev[0].record()
for _ in range(10):
    asp.score_select(step.q_hat, step.k_cache, step.seq_lens, 2048, sel_idx=step.sel_idx, workspace=step.ws_sel, params=step.p_sel)
ev[1].record(); torch.cuda.synchronize()
print("ASP_SCORE_EXP=%s score_select_us=%.1f" % (os.environ.get("ASP_SCORE_EXP", "0"), ev[0].elapsed_time(ev[1]) / 10 * 1000))

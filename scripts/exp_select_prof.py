"""Phase timing of the select kernel (instrumented build, -DASP_PROFILE_SELECT),
config [2]: cycles of CTA thread 0 per phase, averaged per row."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ASYNCSPADE_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build/prof/libasyncspade_prof.so")
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
P = int(os.environ.get("SHARD", "1"))
step = DecodeStep(configs.QWEN3_32B, "cuda", kv_heads=(0, 8 // P))
step.fill_synthetic()
asp.predict_query(step.window, step.q_hat, params=step.p_pred)
L = asp.lib()
buf = (ctypes.c_ulonglong * 8)()
for it in range(3):
    L.asp_select_prof_read(buf)
    asp.score_select(step.q_hat, step.k_cache, step.seq_lens, 2048, sel_idx=step.sel_idx, workspace=step.ws_sel, params=step.p_sel)
    torch.cuda.synchronize()
L.asp_select_prof_read(buf)
names = ["sample", "bracket", "classify", "radix", "emit"]
rows = 512 // P
for n, v in zip(names, buf):
    print(f"{n:12s} {v / rows / 1.93e3:8.2f} us/row")
print("candidates per CTA", buf[6] / rows, " fallback CTAs", buf[7])

"""Phase timing of the predict kernel (instrumented build, -DASP_PROFILE_PREDICT),
config [2]: cycles per warp (row) per phase."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ASYNCSPADE_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build/prof/libasyncspade_prof.so")
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
step = DecodeStep(configs.QWEN3_32B, "cuda")
step.fill_synthetic()
L = asp.lib()
buf = (ctypes.c_ulonglong * 8)()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(3):
    L.asp_predict_prof_read(buf)
    ev[0].record()
    asp.predict_query(step.window, step.q_hat, params=step.p_pred)
    ev[1].record(); torch.cuda.synchronize()
L.asp_predict_prof_read(buf)
rows = 64 * 64
print("predict us", ev[0].elapsed_time(ev[1]) * 1000)
for n, v in zip(["gram", "ridge", "coeffs", "combine"], buf):
    print(f"{n:10s} {v / rows / 1.93e3:8.2f} us/row")

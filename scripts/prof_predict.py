"""Phase profile of the predict kernels (instrumented build, -DASP_PROFILE_PREDICT):
per warp, microseconds from kernel entry to the Gram (0), the solve (1, 2) and
the weighted sum's end (3), at config [2] P = 1 (pair kernel) and the P = 8
shard (split kernel), and high concurrency b512.  Dev tool."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07486_b200 import build as asp_build
os.environ["ASYNCSPADE_LIB"] = os.environ.get("PROF_LIB") or asp_build.build_profiling(
    ["-DASP_PROFILE_PREDICT"], tag="profpred")
import torch
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep

for name, P, warps_per_row in [("qwen3-32b_b64_ctx32k", 1, 0.5), ("qwen3-32b_b64_ctx32k", 8, 2),
                               ("high-conc_b512_ctx4k", 1, 0.5)]:
    cfg = configs.by_name(name)
    step = DecodeStep(cfg, "cuda", kv_heads=(0, cfg.n_kv_heads // P))
    step.fill_synthetic()
    L = asp.lib()
    buf = (ctypes.c_ulonglong * 8)()
    f = lambda: asp.predict_query(step.window, step.q_hat, params=step.p_pred)
    for _ in range(3):
        L.asp_predict_prof_read(buf)
        f()
        torch.cuda.synchronize()
    L.asp_predict_prof_read(buf)
    rows = cfg.batch * cfg.n_q_heads // P
    warps = rows * warps_per_row
    print(f"{name} P={P}: {rows} query rows, {warps:.0f} warps")
    for i, nm in [(0, "window + Gram"), (4, "slice sum (split)"), (1, "solve (+ sync)"),
                  (2, "pdl wait"), (3, "weighted sum + store")]:
        print(f"  {nm:22s} {buf[i] / warps / 1965:8.2f} us per warp")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"  predict call {e0.elapsed_time(e1) / 20 * 1e3:.1f} us (instrumented)")
    del step
    torch.cuda.empty_cache()

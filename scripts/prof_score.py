"""Wait-time profile of the score kernel (instrumented build, -DASP_PROFILE_SCORE):
per CTA, microseconds the TMA producer waits for free stages, the MMA issuer
waits for full stages / free accumulators / B operands and spends issuing, and
epilogue warp 4 waits for accumulators, for GQA group sizes 8 / 16 / 32 and
64-head MQA.  Dev tool."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07486_b200 import build as asp_build
os.environ["ASYNCSPADE_LIB"] = os.environ.get("PROF_LIB") or asp_build.build_profiling(
    ["-DASP_PROFILE_SCORE"], tag="profscore")
import torch
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep

names = {0: "tma: stage empty", 1: "mma: stage full", 2: "mma: accum free", 3: "mma: issuing",
         7: "mma: B operand", 4: "epi(w4): accum full", 6: "kernel (thread 0)"}
cases = [configs.Config(f"g{G}", 2, 16, 8 * G, 8, 128, 32768, 2048, 16) for G in (8, 16, 32)]
cases.append(configs.MQA_64)
for cfg in cases:
    step = DecodeStep(cfg, "cuda")
    step.fill_synthetic()
    asp.predict_query(step.window, step.q_hat, params=step.p_pred)
    L = asp.lib()
    buf = (ctypes.c_ulonglong * 8)()
    f = lambda: asp.score_select(step.q_hat, step.k_cache, step.seq_lens, cfg.top_k,
                                 sel_idx=step.sel_idx, workspace=step.ws_sel, params=step.p_sel)
    for _ in range(3):
        L.asp_score_prof_read(buf)
        f()
        torch.cuda.synchronize()
    L.asp_score_prof_read(buf)
    print(cfg.name, "G =", cfg.group)
    for i in sorted(names):
        print(f"  {names[i]:22s} {buf[i] / 148 / 1965:8.2f} us per CTA")
    del step
    torch.cuda.empty_cache()

"""Phase timing of the predict kernel (instrumented build, -DASP_PROFILE_PREDICT):
cycles per warp per phase, config [2] at P = 1 and at the P = 8 shard.
Fast (pair) kernel phases: gram, ridge, coeffs, combine."""
import ctypes, os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["ASYNCSPADE_LIB"] = os.path.join(ROOT, "build/prof/libasyncspade_prof.so")
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
L = asp.lib()
buf = (ctypes.c_ulonglong * 8)()
for cfg, P in ((configs.QWEN3_32B, 1), (configs.QWEN3_32B, 8), (configs.high_concurrency(1), 1)):
    step = DecodeStep(cfg, "cuda", kv_heads=(0, cfg.n_kv_heads // P))
    step.fill_synthetic()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for it in range(3):
        L.asp_predict_prof_read(buf)
        ev[0].record()
        asp.predict_query(step.window, step.q_hat, params=step.p_pred)
        ev[1].record(); torch.cuda.synchronize()
    L.asp_predict_prof_read(buf)
    warps = cfg.batch * step.n_q // 2
    print(f"{cfg.name} P={P} predict us {ev[0].elapsed_time(ev[1]) * 1000:.1f} (instrumented)")
    for n, v in zip(["gram", "ridge", "coeffs", "combine"], buf):
        print(f"  {n:10s} {v / warps / 1.965e3:8.2f} us/warp")
    del step; torch.cuda.empty_cache()

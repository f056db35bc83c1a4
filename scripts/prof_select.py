"""Phase timing of the select kernel (instrumented build, -DASP_PROFILE_SELECT):
cycles of CTA thread 0 per phase, averaged per CTA, on config [2] at P = 1 and
the P-way shard (SHARD=P).  Dev tool: builds build/prof/libasyncspade_prof.so."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07486_b200 import build as asp_build
_extra = os.environ.get("SEL_DEFINES", "").split()
os.environ["ASYNCSPADE_LIB"] = os.environ.get("PROF_LIB") or asp_build.build_profiling(
    ["-DASP_PROFILE_SELECT", *_extra], tag="prof" + "".join(d.replace("-D", "_") for d in _extra))
print("select defines:", _extra or "(default)")
import torch
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep

for P in [int(x) for x in os.environ.get("SHARDS", "1,8").split(",")]:
    cfg = configs.by_name(os.environ.get("CONFIG", "qwen3-32b_b64_ctx32k"))
    step = DecodeStep(cfg, "cuda", kv_heads=(0, cfg.n_kv_heads // P))
    step.fill_synthetic()
    asp.predict_query(step.window, step.q_hat, params=step.p_pred)
    L = asp.lib()
    buf = (ctypes.c_ulonglong * 8)()
    f = lambda: asp.score_select(step.q_hat, step.k_cache, step.seq_lens, cfg.top_k,
                                 sel_idx=step.sel_idx, workspace=step.ws_sel, params=step.p_sel)
    for it in range(3):
        L.asp_select_prof_read(buf)
        f()
        torch.cuda.synchronize()
    L.asp_select_prof_read(buf)
    names = ["sample", "bracket", "gather", "radix", "emit", "sweep"]
    rows = cfg.batch * cfg.n_kv_heads // P
    mhz = 1.965e3
    print(f"{cfg.name} P={P}: {rows} rows")
    for n, v in zip(names, buf):
        print(f"  {n:10s} {v / rows / mhz:8.2f} us/row (thread 0 of each CTA)")
    print("  candidates per row", buf[6] / rows, " fallback CTAs", buf[7])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"  score_select call {e0.elapsed_time(e1) / 10 * 1e3:.1f} us (instrumented build)")
    # the select kernel alone, on a kept score buffer (scores L2-warm after the first call)
    sc = torch.empty(step.sel_idx.shape[0], step.sel_idx.shape[1], cfg.seq_len, dtype=torch.float32, device="cuda")
    asp.score_select(step.q_hat, step.k_cache, step.seq_lens, cfg.top_k, sel_idx=step.sel_idx,
                     scores=sc, workspace=step.ws_sel, params=step.p_sel)
    ref_idx = step.sel_idx.clone()
    so = lambda: L.asp_select_only(ctypes.byref(step.p_sel), ctypes.c_void_p(sc.data_ptr()),
                                   ctypes.c_void_p(step.seq_lens.data_ptr()),
                                   ctypes.c_void_p(step.sel_idx.data_ptr()), None,
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    for _ in range(3):
        so()
    torch.cuda.synchronize()
    assert torch.equal(step.sel_idx, ref_idx), "select-only differs from score_select"
    e0.record()
    for _ in range(20):
        so()
    e1.record()
    torch.cuda.synchronize()
    print(f"  select alone {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call (20 back-to-back calls)")
    del step, sc
    torch.cuda.empty_cache()

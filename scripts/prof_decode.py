"""Wait-time profile of the decode kernel (instrumented build, -DASP_PROFILE_DECODE):
per CTA, microseconds that producer thread 0 / the MMA thread / softmax thread 0
spend in each barrier wait, on config [2] (P = 1, the P = 8 shard) and the
high-concurrency batch-512 step.  Dev tool."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07486_b200 import build as asp_build
_extra = os.environ.get("DEC_DEFINES", "").split()
os.environ["ASYNCSPADE_LIB"] = asp_build.build_profiling(
    ["-DASP_PROFILE_DECODE", *_extra], tag="profdec" + "".join(d.replace("-D", "_") for d in _extra))
import torch
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep

names = {0: "prod: Q slot empty", 1: "prod: tok slot empty", 2: "prod: stage empty",
         11: "prod: cp.async wait", 3: "mma: stage full", 4: "mma: Q full", 5: "mma: P full",
         6: "mma: O empty", 7: "smx: tok full", 8: "smx: S full", 9: "epi: O full",
         10: "kernel (thread 0)"}
for name, P in [("qwen3-32b_b64_ctx32k", 1), ("qwen3-32b_b64_ctx32k", 8), ("high-conc_b512_ctx4k", 1)]:
    cfg = configs.by_name(name)
    step = DecodeStep(cfg, "cuda", kv_heads=(0, cfg.n_kv_heads // P))
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    L = asp.lib()
    buf = (ctypes.c_ulonglong * 16)()
    f = lambda: asp.sparse_decode(step.q, step.k_cache, step.v_cache, step.seq_lens, step.sel_idx,
                                  out=step.out, workspace=step.ws_dec, params=step.p_dec)
    for _ in range(3):
        L.asp_decode_prof_read(buf)
        f()
        torch.cuda.synchronize()
    L.asp_decode_prof_read(buf)
    ctas = min(148, 10**9)
    print(f"{name} P={P}")
    for i in sorted(names):
        print(f"  {names[i]:22s} {buf[i] / ctas / 1965:8.2f} us per CTA")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"  sparse_decode call {e0.elapsed_time(e1) / 20 * 1e3:.1f} us (instrumented)")
    del step
    torch.cuda.empty_cache()

"""A/B: score_select (or, with AB_CALL=decode, sparse_decode) call time (CUDA events, 20 eager calls after warm-up) for
several builds of the library, on config [2] at P = 1 and the P = 8 shard,
high concurrency b512 and the long-CoT 512k shard.  Dev tool.
usage: python scripts/ab_select.py lib1.so lib2.so ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import os, sys, torch
sys.path.insert(0, %r)
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
res = []
WL = os.environ.get("AB_WORKLOADS", "qwen3-32b_b64_ctx32k:1,qwen3-32b_b64_ctx32k:8,"
                    "high-conc_b512_ctx4k:1,long-cot_b8_ctx524288:8")
for name, shard in ((w.split(":")[0], int(w.split(":")[1])) for w in WL.split(",")):
    cfg = configs.by_name(name)
    st = DecodeStep(cfg, "cuda", kv_heads=(0, cfg.n_kv_heads // shard))
    st.fill_synthetic()
    asp.predict_query(st.window, st.q_hat, params=st.p_pred)
    asp.score_select(st.q_hat, st.k_cache, st.seq_lens, cfg.top_k, sel_idx=st.sel_idx,
                     workspace=st.ws_sel, params=st.p_sel)
    if os.environ.get("AB_CALL") == "predict":
        f = lambda: asp.predict_query(st.window, st.q_hat, params=st.p_pred)
    elif os.environ.get("AB_CALL") == "decode":
        f = lambda: asp.sparse_decode(st.q, st.k_cache, st.v_cache, st.seq_lens, st.sel_idx,
                                      out=st.out, workspace=st.ws_dec, params=st.p_dec)
    else:
        f = lambda: asp.score_select(st.q_hat, st.k_cache, st.seq_lens, cfg.top_k, sel_idx=st.sel_idx,
                                     workspace=st.ws_sel, params=st.p_sel)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    res.append("%%s/P%%d %%.1f" %% (name, shard, e0.elapsed_time(e1) / 20 * 1e3))
    del st; torch.cuda.empty_cache()
print(" | ".join(res))
''' % ROOT
for lib in sys.argv[1:]:
    env = dict(os.environ, ASYNCSPADE_LIB=lib)
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(os.path.basename(os.path.dirname(lib)) or lib, os.environ.get("AB_CALL", "score_select"), "us:",
          r.stdout.strip() or r.stderr[-800:])

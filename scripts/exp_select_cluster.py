"""score_select call time vs forced cluster size (profile build, ASP_SELECT_CLUSTER)
on the P = 8 / P = 4 shards of config [2] and config [1]."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import os, sys, torch
sys.path.insert(0, "%s")
os.environ["ASYNCSPADE_LIB"] = os.path.join("%s", "build/prof/libasyncspade_prof.so")
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
for cfg, P in [(configs.QWEN3_32B, 8), (configs.QWEN3_32B, 4), (configs.QWEN3_32B, 2)]:
    step = DecodeStep(cfg, "cuda", kv_heads=(0, cfg.n_kv_heads // P))
    step.fill_synthetic()
    asp.predict_query(step.window, step.q_hat, params=step.p_pred)
    f = lambda: asp.score_select(step.q_hat, step.k_cache, step.seq_lens, cfg.top_k, sel_idx=step.sel_idx,
                                 workspace=step.ws_sel, params=step.p_sel)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    print(f"C={os.environ.get('ASP_SELECT_CLUSTER')} P={P} score_select {e0.elapsed_time(e1) / 20 * 1e3:9.1f} us", flush=True)
    del step; torch.cuda.empty_cache()
''' % (ROOT, ROOT)
for C in ("1", "2", "4"):
    env = dict(os.environ, ASP_SELECT_CLUSTER=C)
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=120)
    print(r.stdout.strip(), r.stderr.strip()[-300:])

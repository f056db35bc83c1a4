"""score_select call time (CUDA events) on config [2], the long-CoT 512k shard
and high-concurrency b512 -- quick A/B of the select kernel."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
for cfg, kvh in [(configs.QWEN3_32B, None), (configs.long_cot(524288), (0, 1)),
                 (configs.long_cot(32768), (0, 1)), (configs.high_concurrency(512), None)]:
    step = DecodeStep(cfg, "cuda", kv_heads=kvh)
    step.fill_synthetic()
    asp.predict_query(step.window, step.q_hat, params=step.p_pred)
    f = lambda: asp.score_select(step.q_hat, step.k_cache, step.seq_lens, cfg.top_k, sel_idx=step.sel_idx,
                                 workspace=step.ws_sel, params=step.p_sel)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    print(f"{cfg.name:28s} score_select {e0.elapsed_time(e1) / 10 * 1e3:9.1f} us")
    del step; torch.cuda.empty_cache()

"""Is the first decode after select different from later decodes? (debug)"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
step = DecodeStep(configs.QWEN3_8B, "cuda")
step.fill_synthetic()
def dec():
    asp.sparse_decode(step.q, step.k_cache, step.v_cache, step.seq_lens, step.sel_idx, out=step.out, workspace=step.ws_dec, params=step.p_dec)
asp.predict_query(step.window, step.q_hat, params=step.p_pred)
asp.score_select(step.q_hat, step.k_cache, step.seq_lens, step.cfg.top_k, sel_idx=step.sel_idx, workspace=step.ws_sel, params=step.p_sel)
torch.cuda.synchronize()
idx0 = step.sel_idx.clone()
dec(); torch.cuda.synchronize(); a = step.out.clone()
dec(); torch.cuda.synchronize(); b = step.out.clone()
print("sync'd first==second:", torch.equal(a, b), "idx stable:", torch.equal(idx0, step.sel_idx))
step.ws_dec.zero_(); dec(); torch.cuda.synchronize(); c = step.out.clone()
print("after zeroing workspace equal:", torch.equal(a, c))
step.ws_dec.fill_(255); dec(); torch.cuda.synchronize(); d = step.out.clone()
print("after NaN-filling workspace equal:", torch.equal(a, d), "max diff", (a - d).abs().max().item())
torch.cuda.empty_cache()
# L2 flush then decode
junk = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda"); junk.fill_(1); torch.cuda.synchronize()
dec(); torch.cuda.synchronize(); e = step.out.clone()
print("after L2 flush equal:", torch.equal(a, e), "max diff", (a - e).abs().max().item(), "rows differing", int(((a - e).abs().amax(dim=2) > 0).sum()))

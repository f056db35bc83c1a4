"""A small composed step of every entry point, for compute-sanitizer runs:
append -> predict -> score_select (dense and paged) -> decode -> gather ->
quest, on a ragged two-sequence batch; then full steps at G = 16 and G = 32,
the round-2 kernels (head-dim-split predict, G = 64 tensor-core score,
CUDA-core score / decode for absorbed MLA and 128-head MQA, single-chunk
direct output, head-major output, window-less append), and session 3's
one-item decode rows and cluster-split long rows."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
cfg = configs.QWEN3_8B.with_(batch=2, seq_len=1024, top_k=128)
st = DecodeStep(cfg, "cuda", n_fresh=1)
st.fill_synthetic()
st.seq_lens.copy_(torch.tensor([1024, 700], dtype=torch.int32))
g = torch.Generator().manual_seed(1)
st.append(torch.randn(2, 32, 128, generator=g).cuda(),
          torch.randn(2, 8, 128, generator=g).to(torch.bfloat16).cuda(),
          torch.randn(2, 8, 128, generator=g).to(torch.bfloat16).cuda(),
          torch.tensor([1023, 699], dtype=torch.int32, device="cuda"))
st.run()
pool, bt = asp.page_pool(st.k_cache, 16, torch.Generator().manual_seed(2))
vpool, _ = asp.page_pool(st.v_cache, 16, torch.Generator().manual_seed(2))
idx = asp.score_select_paged(st.q_hat, pool, bt, st.seq_lens, cfg.top_k, cfg.seq_len)
asp.sparse_decode_paged(st.q, pool, vpool, bt, st.seq_lens, idx, cfg.seq_len, n_fresh=1)
asp.gather_filtered(st.k_cache, st.v_cache, st.seq_lens, st.sel_idx, n_fresh=1)
meta = asp.quest_summarize(st.k_cache, st.seq_lens, 16, cfg.top_k, 32)
asp.quest_select(st.q_hat, meta, st.k_cache, st.seq_lens, cfg.top_k, 16)
# GQA group 16 and 32-head MQA (the largest P / Q operands and TMEM layouts)
for G, hkv in ((16, 2), (32, 1)):
    c2 = configs.Config(f"g{G}", 0, 2, G * hkv, hkv, 128, 2048, 256, 16)
    s2 = DecodeStep(c2, "cuda", n_fresh=1)
    s2.fill_synthetic()
    s2.run()
    flags = int(s2.dev_flags.item())
    assert flags == 0, flags
# round 2: MQA 64 / 128 heads, absorbed MLA (values from the key rows), a
# single-chunk decode (k + n_fresh <= 256), head-major output, window-less append
for c2 in (configs.Config("mqa64", 0, 2, 64, 1, 128, 2048, 256, 16),
           configs.Config("mqa128", 0, 2, 128, 1, 128, 2048, 128, 16),
           configs.Config("mla4", 0, 2, 4, 1, 576, 1024, 128, 16, v_head_dim=512)):
    s2 = DecodeStep(c2, "cuda", n_fresh=1, out_head_major=c2.name == "mqa64")
    s2.fill_synthetic()
    s2.run()
    flags = int(s2.dev_flags.item())
    assert flags == 0, flags
# session 3: a one-item 3-tile decode row (k + n_fresh = 257), and long rows
# split over 8-CTA clusters with 64k-key segments (DSMEM reduce-scatter merges,
# 64k direct emission) feeding the staged-scale combine (129 chunks per row)
for c2 in (configs.Config("onei", 0, 2, 16, 2, 128, 2048, 256, 16),
           configs.Config("longrow", 0, 5, 2, 1, 128, 524288, 32768, 16)):
    s2 = DecodeStep(c2, "cuda", n_fresh=1)
    s2.fill_synthetic()
    s2.run()
    flags = int(s2.dev_flags.item())
    assert flags == 0, flags
    del s2
q_only = torch.empty(2, 32, 128, dtype=torch.bfloat16, device="cuda")
asp.append(torch.randn(2, 32, 128, generator=g).cuda(), None, 0, q_cur=q_only)
torch.cuda.synchronize()
print("sanitize-small ok, flags", int(st.dev_flags.item()))

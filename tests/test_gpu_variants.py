"""GPU parity for the NEXT-3 attention variants:
absorbed MLA -- one KV head whose key is the 576-dim latent (+ rope) and whose
value is its first 512 dims -- and multi-query attention with 64 / 128 query
heads on one KV head, through every step of the path (predict at D = 576,
score + top-k, sparse decode with V read from the key rows), against the
oracle on the same seeded inputs (tolerances: tests/parity_util.py)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import build as asp_build
from paper_2510_07486_b200 import configs, synth
from paper_2510_07486_b200.step import DecodeStep
from parity_util import ATTN_RTOL, Q_HAT_RTOL, check_selection, rel_inf_err, rows_sample

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _built():
    asp_build.build()
    asp.lib()


def _dev(bits):
    return torch.from_numpy(bits.view(np.int16).copy()).to(DEV).view(torch.bfloat16)


@pytest.mark.parametrize("D,G", [(576, 1), (576, 4), (576, 16), (128, 64), (128, 128),
                                 (64, 64), (256, 8)])
def test_score_select_wide_shapes(D, G):
    """score + top-k for shapes outside the tensor-core stream: band-rule
    index sets and scores within 1e-5 of the oracle's, ragged rows."""
    B, Hkv, L, k = 2, 1 if G >= 16 else 2, 3000, 190
    lens = [3000, 2011]
    K = synth.kv_cache(900 + D + G, synth.STREAM_K, B, Hkv, L, D)
    qh = (np.random.default_rng(D * G).standard_normal((B, Hkv * G, D)) * 0.3).astype(np.float32)
    sl = torch.tensor(lens, dtype=torch.int32, device=DEV)
    scores = torch.full((B, Hkv, L), np.nan, dtype=torch.float32, device=DEV)
    flags = torch.zeros(1, dtype=torch.int32, device=DEV)
    idx = asp.score_select(torch.from_numpy(qh).to(DEV), _dev(K), sl, k, scores=scores,
                           dev_flags=flags).cpu().numpy()
    assert int(flags.item()) == 0
    so, _ = oracle.score(qh, K, lens)
    sg = scores.cpu().numpy()
    for b in range(B):
        for h in range(Hkv):
            n = lens[b]
            assert np.abs(sg[b, h, :n] - so[b, h, :n]).max() <= 1e-5 * np.abs(so[b, h, :n]).max()
            check_selection(idx[b, h], so[b, h], n, k)


@pytest.mark.parametrize("D,Dv,G,n_fresh,Hkv", [(576, 512, 16, 0, 1), (576, 512, 16, 1, 1),
                                                (576, 512, 1, 1, 1), (128, 128, 64, 1, 1),
                                                (128, 128, 128, 0, 1), (64, 64, 64, 3, 1),
                                                (128, 128, 64, 1, 2)])
def test_decode_wide_shapes(D, Dv, G, n_fresh, Hkv):
    """Sparse decode for absorbed MLA (V = the first 512 dims of the key rows,
    one cache) and 64 / 128 query heads per KV head -- on the tensor cores as
    virtual KV heads when there is one KV head (MQA), on the CUDA cores with
    two: within 2e-3 of the oracle, 3 chunks with -1 padding and the fresh
    tail."""
    rng = np.random.default_rng(D + G + n_fresh + Hkv)
    B, L, k = 2, 1500, 600
    lens = [1500, 900]
    K = synth.kv_cache(77 + D, synth.STREAM_K, B, Hkv, L, D)
    mla = Dv < D
    V = np.ascontiguousarray(K[..., :Dv]) if mla else synth.kv_cache(77 + D, synth.STREAM_V, B, Hkv, L, D)
    _, q = synth.query_trace(5 + G, B, Hkv * G, 2, D)
    idx = np.full((B, Hkv, k), -1, np.int32)
    for b in range(B):
        m = min(k - 7, lens[b])
        for h in range(Hkv):
            idx[b, h, :m] = np.sort(rng.choice(lens[b], m, replace=False))
    Kd = _dev(K)
    Vd = Kd if mla else _dev(V)
    p = asp.decode_params(_dev(q), Kd, Vd, k, n_fresh, v_head_dim=Dv if mla else 0)
    out = asp.sparse_decode(_dev(q), Kd, Vd, torch.tensor(lens, dtype=torch.int32, device=DEV),
                            torch.from_numpy(idx).to(DEV), params=p).cpu().numpy()
    assert out.shape == (B, Hkv * G, Dv)
    ref = oracle.sparse_decode(q, K, V, idx, lens, n_fresh)
    assert rel_inf_err(out, ref) <= ATTN_RTOL


@pytest.mark.parametrize("D", [576, 256])
def test_predict_wide_head_dim(D):
    """a1 at the absorbed-MLA query width (576) and 256: the generic kernel,
    every assembly mode, against the oracle."""
    for flags in (0, asp.ASSEMBLY_SINGLE, asp.ASSEMBLY_PER_WINDOW, asp.SIGN_NEGATED):
        win, _ = synth.query_trace(synth.base_seed(3) + D, 3, 5, 16, D)
        g = asp.predict_query(torch.from_numpy(win).to(DEV), flags=flags)
        ref, cond = oracle.predict(win, 1e-2, flags)
        assert cond == 0
        assert rel_inf_err(g.cpu().numpy(), ref) <= Q_HAT_RTOL


@pytest.mark.parametrize("name", ["mla16", "mqa64"])
def test_step_variants_against_oracle(name):
    """The whole step (predict -> score -> top-k -> decode) for the absorbed-MLA
    and 64-head MQA configs (reduced batch / context), every row against the
    oracle, chained, plus the unchained Eq. 1 overlap."""
    base = configs.MLA_16 if name == "mla16" else configs.MQA_64
    cfg = base.with_(batch=3, seq_len=4096, top_k=256)
    step = DecodeStep(cfg, DEV, n_fresh=1)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    assert int(step.dev_flags.item()) == 0
    seed = synth.base_seed(cfg.index)
    dv = cfg.v_head_dim or cfg.head_dim

    def kv(b, h):
        Kr = synth.kv_rows(seed, synth.STREAM_K, b, h, 0, cfg.seq_len, cfg.n_kv_heads,
                           cfg.seq_len, cfg.head_dim)
        Vr = (np.ascontiguousarray(Kr[:, :dv]) if dv < cfg.head_dim else
              synth.kv_rows(seed, synth.STREAM_V, b, h, 0, cfg.seq_len, cfg.n_kv_heads,
                            cfg.seq_len, cfg.head_dim))
        return Kr, Vr

    from test_gpu_parity import _oracle_row_checks
    ov = []
    _oracle_row_checks(step, range(cfg.batch * cfg.n_kv_heads), n_fresh=1, overlap=ov, kv_rows=kv)
    assert np.mean(ov) >= 0.99, ov

"""GPU parity, round 2: the a5 pipeline step by step against the oracle,
structured (needle / sink) keys at config [2]'s shape, reading R14's float
edge cases (NaN keys, signed zeros), and the exactly-linear invariant of the
predictor (R17) -- all through the C ABI, all against oracle/ on the same
seeded inputs (tolerances: tests/parity_util.py)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import build as asp_build
from paper_2510_07486_b200 import configs, synth
from paper_2510_07486_b200.pipeline import AsyncPipeline
from paper_2510_07486_b200.step import DecodeStep
from parity_util import ATTN_RTOL, Q_HAT_RTOL, check_selection, rel_inf_err, rows_sample

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _built():
    asp_build.build()
    asp.lib()


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _dev_bf16(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(bits.view(np.int16).copy()).to(DEV).view(torch.bfloat16)


# ----------------------------------------------------------------------------- a5 vs oracle
@pytest.mark.parametrize("mode", ["pipelined", "serial"])
def test_async_pipeline_each_step_matches_oracle(mode):
    """a5 (the Cache Rank 'enqueues the query state to the sliding
    window, then proactively performs token-level KV cache filtering required
    for the next decoding step'): T steps of the pipeline, each pushing a new
    query and K/V row, mirrored on the host.  Per step t, on EVERY row:
      * out(t) == oracle attention over the indices the GPU used at t plus the
        fresh token (n_fresh = 1), on the host cache after push(t);
      * q_hat(t+1) == oracle.predict on the host window after push(t) (the
        ring has advanced: logical order follows ring_start);
      * idx(t+1) obeys the band rule against the oracle's scores of the GPU
        q_hat (chained), and the unchained oracle selection overlaps it
        (Eq. 1) >= 0.999 on average."""
    cfg = configs.high_concurrency(4)               # Qwen3-8B shape, 4k context, k = 256
    B, Hq, Hkv, D, L, W, k = (cfg.batch, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim,
                              cfg.seq_len, cfg.window, cfg.top_k)
    G = cfg.group
    T = 5
    g = torch.Generator().manual_seed(23)
    qts = [torch.randn(B, Hq, D, generator=g) * 0.5 for _ in range(T)]
    kvs = [torch.randn(2, B, Hkv, D, generator=g).to(torch.bfloat16) for _ in range(T)]

    step = DecodeStep(cfg, DEV, n_fresh=1)
    step.fill_synthetic()
    pipe = AsyncPipeline(step, forward_bytes=32 << 20)
    seed = synth.base_seed(cfg.index)
    win, q_bits = synth.query_trace(seed, B, Hq, W, D)
    ring = np.array(win)                             # physical ring, ring_start 0
    rs = 0
    K = synth.kv_cache(seed, synth.STREAM_K, B, Hkv, L, D)
    V = synth.kv_cache(seed, synth.STREAM_V, B, Hkv, L, D)
    lens = [L] * B
    overlaps = []
    for t in range(T):
        (pipe.run_step if mode == "pipelined" else pipe.run_step_serial)(
            qts[t].to(DEV), kvs[t].to(DEV))
        pipe.drain()
        torch.cuda.synchronize()
        idx_used = pipe.idx[t % 2].cpu().numpy()
        idx_next = pipe.idx[(t + 1) % 2].cpu().numpy()
        qh_g = step.q_hat.cpu().numpy()
        out_g = step.out.cpu().numpy()
        # host mirror of a0 (asyncspade_append): q_t into the ring slot, its bf16
        # rounding is the current query, the K / V rows at seq_len - 1
        ring[:, :, rs] = qts[t].numpy()
        rs = (rs + 1) % W
        q_bits = synth.f32_to_bf16_bits(qts[t].numpy())
        K[:, :, L - 1] = _bits(kvs[t][0])
        V[:, :, L - 1] = _bits(kvs[t][1])
        assert step.ring_start == rs
        # decode(t) on the indices the GPU used at step t
        o_or = oracle.sparse_decode(q_bits, K, V, idx_used, lens, n_fresh=1)
        assert rel_inf_err(out_g, o_or) <= ATTN_RTOL, t
        # q_hat for t+1 from the advanced ring
        qh_or, cond = oracle.predict(ring, step.eps, step.flags, rs)
        assert cond == 0
        assert rel_inf_err(qh_g, qh_or) <= Q_HAT_RTOL, t
        # selection for t+1: chained band rule on every row, unchained overlap
        s_ch, _ = oracle.score(qh_g, K, lens)
        s_un, _ = oracle.score(qh_or, K, lens)
        i_un, _ = oracle.select(s_un, k)
        for b in range(B):
            for h in range(Hkv):
                check_selection(idx_next[b, h], s_ch[b, h], L, k)
                overlaps.append(len(np.intersect1d(idx_next[b, h], i_un[b, h])) / k)
    assert np.mean(overlaps) >= 0.999, np.mean(overlaps)
    # the selections really moved with the pushed queries
    assert not np.array_equal(pipe.idx[0].cpu().numpy(), pipe.idx[1].cpu().numpy())


# ----------------------------------------------------------------------------- structured keys
def test_step_qwen3_32b_needles_and_sink():
    """SURVEY §8(d) structured inputs at config [2]'s full shape: 32 heavy-hitter
    needles per row and an attention sink at token 0, planted along the
    newest window query of the KV head's first q head.  The 32-row subset is
    checked chained against the oracle on the same planted keys, and every
    needle and the sink must be selected on every row (they out-score the
    1/16 budget's threshold by >10 sigma)."""
    cfg = configs.QWEN3_32B
    step = DecodeStep(cfg, DEV)
    step.fill_synthetic()
    seed = synth.base_seed(cfg.index)
    synth.apply_structure_device(step.k_cache, seed, cfg.seq_len, cfg.n_kv_heads, cfg.group,
                                 cfg.n_q_heads, cfg.window)
    step.run()
    torch.cuda.synchronize()
    assert int(step.dev_flags.item()) == 0
    idx = step.sel_idx.cpu().numpy()
    for b in range(cfg.batch):
        for h in range(cfg.n_kv_heads):
            need = np.concatenate([[0], synth.needle_positions(seed, b, h, cfg.seq_len)])
            assert np.isin(need, idx[b, h]).all(), (b, h)

    def kv(b, h):
        Ks = synth.structured_kv_rows(seed, b, h, cfg.seq_len, cfg.n_kv_heads, cfg.seq_len,
                                      cfg.head_dim, cfg.group, cfg.n_q_heads, cfg.window)
        Vs = synth.kv_rows(seed, synth.STREAM_V, b, h, 0, cfg.seq_len, cfg.n_kv_heads,
                           cfg.seq_len, cfg.head_dim)
        return Ks, Vs

    # the device planting is the host planting, bit for bit (two sampled rows)
    for b, h in ((0, 0), (37, 5)):
        np.testing.assert_array_equal(_bits(step.k_cache[b, h]), kv(b, h)[0])
    from test_gpu_parity import _oracle_row_checks
    ov = []
    _oracle_row_checks(step, rows_sample(cfg.batch * cfg.n_kv_heads, 32, seed=9), overlap=ov,
                       kv_rows=kv)
    assert np.mean(ov) >= 0.999, np.mean(ov)
    del step
    torch.cuda.empty_cache()


# ----------------------------------------------------------------------------- R14
def _select_on(K, q, lens, k, G):
    Kd = _dev_bf16(K)
    sl = torch.tensor(lens, dtype=torch.int32, device=DEV)
    flags = torch.zeros(1, dtype=torch.int32, device=DEV)
    idx = asp.score_select(torch.from_numpy(q).to(DEV), Kd, sl, k, dev_flags=flags)
    return idx.cpu().numpy(), int(flags.item())


@pytest.mark.parametrize("L,k", [(1000, 37), (40000, 2048), (131072, 8192)])
def test_r14_nan_keys_rank_last_and_flag(L, k):
    """R14: a key row holding a NaN gives a NaN score, which ranks below every
    number: it is selected only when a row has fewer than k non-NaN tokens (the
    lowest-index NaNs then fill it, as in the oracle's sort), and the call sets
    ASP_FLAG_NONFINITE.  Row 0: a few NaN keys; row 1: all but k/2 NaN;
    row 2: NaN keys clustered where the top scores would be.  Covers the
    single-CTA and cluster-split select paths."""
    rng = np.random.default_rng(L + k)
    B, Hkv, G, D = 3, 1, 4, 128
    K = synth.kv_cache(1234 + L, synth.STREAM_K, B, Hkv, L, D)
    q = (rng.standard_normal((B, Hkv * G, D)) * 0.5).astype(np.float32)
    nan = np.uint16(0x7FC0)
    K[0, 0, rng.choice(L, 17, replace=False), 3] = nan
    keep = rng.choice(L, k // 2, replace=False)
    mask = np.ones(L, bool)
    mask[keep] = False
    K[1, 0, mask, 5] = nan
    s_clean, _ = oracle.score(q, K.copy(), [L] * B)
    top = np.argsort(-s_clean[2, 0])[: k // 3]
    K[2, 0, top, 0] = nan
    idx, flags = _select_on(K, q, [L] * B, k, G)
    assert flags & asp.FLAG_NONFINITE
    s_or, cond = oracle.score(q, K, [L] * B)
    ref, _ = oracle.select(s_or, k)
    for b in range(B):
        nan_b = np.isnan(s_or[b, 0])
        assert nan_b.any()
        if b == 1:                                   # fewer than k finite tokens: exact
            np.testing.assert_array_equal(idx[b, 0], ref[b, 0])
            assert nan_b[idx[b, 0]].sum() == k - k // 2
        else:                                        # no NaN is taken while numbers remain
            assert not nan_b[idx[b, 0]].any()
            check_selection(idx[b, 0], np.where(nan_b, -np.inf, s_or[b, 0]), L, k)


def test_r14_signed_zero_scores_tie_lower_index_wins():
    """R14: -0.0 and +0.0 scores tie (the lower index wins, R9).  Zero keys
    (+0.0 and -0.0 bf16 rows) score exactly +-0 whatever the query; 30 keys
    score positive, the rest negative, and k = 37 falls inside the zero
    block -- the selection must be the 30 positives plus the 7 lowest-index
    zero keys, exactly the oracle's."""
    rng = np.random.default_rng(77)
    B, Hkv, G, D, L, k = 2, 1, 2, 64, 2000, 37
    q = np.abs(rng.standard_normal((B, G, D))).astype(np.float32) + 0.1   # positive query
    base = np.abs(rng.standard_normal((B, Hkv, L, D))).astype(np.float32) + 0.1
    K = synth.f32_to_bf16_bits(-base)                                   # negative scores
    pos = rng.choice(L, 30, replace=False)
    K[:, :, pos] = synth.f32_to_bf16_bits(base[:, :, pos])             # 30 positive scores
    zeros = np.setdiff1d(rng.choice(L, 200, replace=False), pos)
    K[:, :, zeros] = np.where(rng.random((B, Hkv, len(zeros), 1)) < 0.5, 0x0000,
                              0x8000).astype(np.uint16)                  # +0.0 / -0.0 rows
    q[1] = -q[1]                                      # batch 1: the products flip sign
    K[1] = K[1] ^ np.uint16(0x8000)                   # ... and so do the keys: same order
    idx, flags = _select_on(K, q, [L] * B, k, G)
    assert flags == 0
    s_or, _ = oracle.score(q, K, [L] * B)
    ref, _ = oracle.select(s_or, k)
    for b in range(B):
        np.testing.assert_array_equal(idx[b, 0], ref[b, 0])
        exp = np.sort(np.concatenate([pos, np.sort(zeros)[: k - 30]]))
        np.testing.assert_array_equal(idx[b, 0], exp)


# ----------------------------------------------------------------------------- R17 on the GPU
def test_predict_exactly_linear_recurrence_gpu():
    """North star 'the regressor reproduces exactly-linear query sequences'
    (reading R17): NORM_NONE + SINGLE + absolute eps = 1e-12 on an exact
    order-(W-1) recurrence with dyadic coefficients and small-integer starts
    (every value exact in fp32) -- the GPU's q_hat equals the recurrence's
    next element within 1e-6 relative (fp64 Gram + solve, fp32 output)."""
    rng = np.random.default_rng(31)
    for W, D in ((5, 64), (8, 128), (4, 128)):
        n = W - 1
        rows = []
        nxt = []
        while len(rows) < 24:
            c = rng.choice([-0.5, -0.25, 0.25, 0.5, 0.125], size=n)
            seq = [rng.integers(-3, 4, D).astype(np.float64) for _ in range(n)]
            for _ in range(2):
                seq.append(sum(c[i] * seq[-1 - i] for i in range(n)))
            w = np.array(seq[:W], np.float32)
            if not np.array_equal(w.astype(np.float64), np.array(seq[:W])):
                continue
            H = np.array(seq[:n])
            if np.linalg.matrix_rank(H) < n:
                continue
            rows.append(w)
            nxt.append(seq[W])
        win = np.stack(rows)[None]                               # [1, 24, W, D]
        flags = asp.ASSEMBLY_SINGLE | asp.NORM_NONE | asp.EPS_ABSOLUTE
        g = asp.predict_query(torch.from_numpy(win).to(DEV), eps=1e-12, flags=flags)
        g = g.cpu().numpy()[0].astype(np.float64)
        ref = np.array(nxt)
        err = np.abs(g - ref).max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1.0)
        assert err.max() <= 1e-6, (W, err.max())
        qh_or, cond = oracle.predict(win, 1e-12, flags)
        assert cond == 0
        assert rel_inf_err(g[None], qh_or) <= 1e-6

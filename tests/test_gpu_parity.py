"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, on the
same seeded inputs, element by element.  Tolerances: tests/parity_util.py
(BASELINE.json north star).  Chained parity feeds the oracle the GPU's own
upstream output (GPU q_hat into the oracle's scorer, GPU idx into the
oracle's decode) so a legitimately different near-tie upstream cannot flip
a downstream check."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import build as asp_build
from paper_2510_07486_b200 import configs, synth
from paper_2510_07486_b200.step import DecodeStep
from parity_util import (ATTN_RTOL, Q_HAT_RTOL, check_selection, rel_inf_err, rows_sample)

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _built():
    asp_build.build()
    asp.lib()


def to_dev_bf16(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(bits.view(np.int16).copy()).to(DEV).view(torch.bfloat16)


def from_dev_bf16(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


# ----------------------------------------------------------------------------- inputs
def test_device_generator_matches_host():
    """The device generator (csrc/synth.cu) reproduces synth.py bit for bit,
    including a head shard (b0/h0 offsets)."""
    seed = synth.base_seed(1)
    k = torch.empty(2, 3, 40, 128, dtype=torch.bfloat16, device=DEV)
    synth.fill_kv_device(k, seed, synth.STREAM_K, 0, 5, 8)
    host = synth.kv_cache(seed, synth.STREAM_K, 2, 3, 40, 128, h0=5, n_kv_heads_global=8)
    np.testing.assert_array_equal(from_dev_bf16(k), host)
    win = torch.empty(2, 4, 16, 64, dtype=torch.float32, device=DEV)
    q = torch.empty(2, 4, 64, dtype=torch.bfloat16, device=DEV)
    synth.fill_query_device(win, q.view(torch.int16), seed, 0, 4, 8)
    hw, hq = synth.query_trace(seed, 2, 8, 16, 64, h0=4, head_slice=4)
    np.testing.assert_array_equal(win.cpu().numpy(), hw)
    np.testing.assert_array_equal(from_dev_bf16(q), hq)


# ----------------------------------------------------------------------------- a1 predict
PRED_FLAGS = [0, asp.ASSEMBLY_SINGLE, asp.ASSEMBLY_PER_WINDOW, asp.DOUBLE_SOFTMAX,
              asp.SIGN_NEGATED, asp.EPS_ABSOLUTE, asp.ASSEMBLY_SINGLE | asp.NORM_NONE]


@pytest.mark.parametrize("flags", PRED_FLAGS)
@pytest.mark.parametrize("shape", [(1, 2, 4, 64), (32, 32, 16, 128), (3, 5, 32, 64), (2, 3, 2, 128),
                                   (3, 5, 9, 128), (1, 3, 8, 64), (7, 3, 17, 128),
                                   # >= 8 x SMs rows: the two-rows-per-warp kernel (fewer
                                   # rows take the head-dim-split kernel)
                                   (40, 32, 16, 128), (37, 33, 9, 64), (41, 29, 5, 128)])
def test_predict_parity(flags, shape):
    B, Hq, W, D = shape
    win, _ = synth.query_trace(synth.base_seed(1) + W, B, Hq, W, D)
    eps = 1e-2 if not flags & asp.EPS_ABSOLUTE else 0.5
    for ring in (0, W // 2):
        phys = np.roll(win, ring, axis=2)        # logical j at physical (ring + j) % W
        g = asp.predict_query(torch.from_numpy(phys).to(DEV), eps=eps, flags=flags,
                              ring_start=ring)
        ref, cond = oracle.predict(phys, eps, flags, ring)
        assert cond == 0
        err = rel_inf_err(g.cpu().numpy(), ref)
        assert err <= Q_HAT_RTOL, err


def test_predict_special_cases_on_gpu():
    """Constant window -> exact; W = 1 passthrough; NaN -> flag 1 +
    passthrough; not-PD (negative absolute eps on a zero history) -> flag 2."""
    q = np.random.default_rng(0).standard_normal(128).astype(np.float32)
    const = np.broadcast_to(q, (4, 3, 16, 128)).copy()
    g = asp.predict_query(torch.from_numpy(const).to(DEV)).cpu().numpy()
    assert np.array_equal(g, np.broadcast_to(q, (4, 3, 128)))
    w1 = np.random.default_rng(1).standard_normal((2, 2, 1, 64)).astype(np.float32)
    assert np.array_equal(asp.predict_query(torch.from_numpy(w1).to(DEV)).cpu().numpy(), w1[:, :, 0])
    bad = np.ones((1, 2, 4, 64), np.float32)
    bad[0, 1, 2, 5] = np.nan
    flags = torch.zeros(1, dtype=torch.int32, device=DEV)
    g = asp.predict_query(torch.from_numpy(bad).to(DEV), dev_flags=flags).cpu().numpy()
    assert flags.item() & asp.FLAG_NONFINITE
    assert np.array_equal(g[0, 1], bad[0, 1, 3]) and np.array_equal(g[0, 0], bad[0, 0, 3])
    z = np.zeros((1, 1, 4, 64), np.float32)
    z[0, 0, 3] = np.arange(64)
    flags.zero_()
    g = asp.predict_query(torch.from_numpy(z).to(DEV), eps=-1.0, flags=asp.EPS_ABSOLUTE,
                          dev_flags=flags).cpu().numpy()
    assert flags.item() & asp.FLAG_NOT_PD and np.array_equal(g[0, 0], z[0, 0, 3])


# ----------------------------------------------------------------------------- a2+a3 select
def _score_select_case(B, Hq, Hkv, D, L, k, seq_lens, seed, kv=None, agg=asp.AGG_MAX):
    rng = np.random.default_rng(seed)
    K = kv if kv is not None else synth.kv_cache(seed, synth.STREAM_K, B, Hkv, L, D)
    qh = (rng.standard_normal((B, Hq, D)) * 0.7).astype(np.float32)
    Kd = to_dev_bf16(K)
    sl = torch.tensor(seq_lens, dtype=torch.int32, device=DEV)
    scores = torch.full((B, Hkv, L), np.nan, dtype=torch.float32, device=DEV)
    flags = torch.zeros(1, dtype=torch.int32, device=DEV)
    idx = asp.score_select(torch.from_numpy(qh).to(DEV), Kd, sl, k, scores=scores,
                           aggregation=agg, dev_flags=flags)
    idx2 = asp.score_select(torch.from_numpy(qh).to(DEV), Kd, sl, k, aggregation=agg)
    assert torch.equal(idx, idx2), "scores-buffer and workspace paths must agree"
    s_or, _ = oracle.score(qh, K, seq_lens, agg)
    return idx.cpu().numpy(), scores.cpu().numpy(), s_or, int(flags.item())


@pytest.mark.parametrize("G", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("D", [64, 128])
def test_score_select_parity_small(G, D):
    B, Hkv, L, k = 3, 2, 1000, 37
    seq_lens = [1000, 777, 256]
    idx, sg, so, flags = _score_select_case(B, Hkv * G, Hkv, D, L, k, seq_lens, 100 + G + D)
    assert flags == 0
    for b in range(B):
        for h in range(Hkv):
            n = seq_lens[b]
            smax = np.abs(so[b, h, :n]).max()
            assert np.abs(sg[b, h, :n] - so[b, h, :n]).max() <= 1e-5 * smax
            check_selection(idx[b, h], so[b, h], n, k)


def test_score_select_sum_aggregation():
    idx, sg, so, _ = _score_select_case(2, 8, 2, 128, 513, 40, [513, 300], 7, agg=asp.AGG_SUM)
    for b, n in enumerate([513, 300]):
        for h in range(2):
            check_selection(idx[b, h], so[b, h], n, 40)


def test_score_select_short_rows_and_extremes():
    """R13 short rows (len < k, len == k, len == 0), k = 1, ragged tail."""
    B, Hkv, G, D, L = 5, 1, 2, 64, 300
    seq_lens = [300, 20, 16, 0, 299]
    idx, _, so, flags = _score_select_case(B, Hkv * G, Hkv, D, L, 16, seq_lens, 11)
    assert flags & asp.FLAG_SHORT_ROW
    for b in range(B):
        check_selection(idx[b, 0], so[b, 0], seq_lens[b], 16)
    idx1, _, so1, _ = _score_select_case(2, 2, 1, 64, 300, 1, [300, 5], 12)
    for b, n in enumerate([300, 5]):
        assert idx1[b, 0, 0] == int(np.argmax(so1[b, 0, :n]))


def test_score_select_exact_ties_lower_index_wins():
    """R9: keys drawn from a 16-row codebook -> massive exact ties; equal keys
    must give equal GPU scores and the lowest indices must win, exactly as in
    the oracle's brute-force sort."""
    rng = np.random.default_rng(21)
    B, Hkv, G, D, L, k = 2, 2, 4, 128, 4096, 700
    book = synth.f32_to_bf16_bits(rng.standard_normal((16, D)).astype(np.float32))
    K = book[rng.integers(0, 16, (B, Hkv, L))]
    idx, sg, so, _ = _score_select_case(B, Hkv * G, Hkv, D, L, k, [L, L - 3], 22, kv=K)
    ref, _ = oracle.select(so, k, np.array([[L, L], [L - 3, L - 3]]))
    np.testing.assert_array_equal(idx, ref)


def test_score_select_all_equal_keys():
    K = np.zeros((1, 1, 2048, 64), np.uint16)
    idx, _, _, _ = _score_select_case(1, 8, 1, 64, 2048, 100, [2048], 3, kv=K)
    np.testing.assert_array_equal(idx[0, 0], np.arange(100))


def test_score_select_long_row_global_path():
    """Rows longer than the shared-memory key cache (40,960 tokens) take the
    L2-streaming path."""
    B, Hkv, G, D, L, k = 1, 1, 8, 128, 65536, 4096
    idx, _, so, _ = _score_select_case(B, Hkv * G, Hkv, D, L, k, [L - 11], 31)
    check_selection(idx[0, 0], so[0, 0], L - 11, k)


@pytest.mark.parametrize("B,L,k", [(1, 131072, 8192), (3, 65536, 4096), (2, 40962, 2560),
                                   (1, 9001, 700), (5, 8192, 512)])
def test_score_select_cluster_split_rows(B, L, k):
    """Rows split over thread-block clusters (C = 2..16 CTAs, chosen from the
    row length and the row count) and the small-CTA path: exact sets; ragged
    lengths put the row end inside a cluster segment."""
    lens = [L - 37 * b for b in range(B)]
    idx, _, so, _ = _score_select_case(B, 8, 1, 128, L, k, lens, 60 + B)
    for b in range(B):
        check_selection(idx[b, 0], so[b, 0], lens[b], k)


def test_score_select_64k_cluster_segments():
    """Long rows over 8-CTA clusters with 64k-key segments (the sel1024w
    instantiation: 64k-key direct emission rounds, DSMEM reduce-scatter
    histogram merges, the bracket-relative radix): exact sets on ragged rows
    whose ends fall inside a segment, and on all-equal keys (every candidate
    list overflows: the exact all-keys radix must give the lowest indices)."""
    B, L, k = 5, 524288, 32768
    lens = [L, L - 37, L - 70001, 300000, 65537]
    idx, _, so, _ = _score_select_case(B, 1, 1, 64, L, k, lens, 91)
    for b in range(B):
        check_selection(idx[b, 0], so[b, 0], lens[b], k)
    K = np.zeros((B, 1, L, 64), np.uint16)
    idx, _, _, _ = _score_select_case(B, 1, 1, 64, L, k, lens, 92, kv=K)
    for b in range(B):
        np.testing.assert_array_equal(idx[b, 0], np.arange(k))


def test_score_select_uncached_longest_rows():
    """Rows beyond 16 x 40,960 tokens: the cluster streams keys from L2."""
    L, k = 720896, 45056
    idx, _, so, _ = _score_select_case(1, 8, 1, 128, L, k, [L - 5], 77)
    check_selection(idx[0, 0], so[0, 0], L - 5, k)


def test_score_select_all_equal_keys_long_row():
    """Massive exact ties on a cluster-split row: the candidate list overflows
    and the exact fallback must still give the lowest indices."""
    K = np.zeros((1, 1, 65536, 64), np.uint16)
    idx, _, _, _ = _score_select_case(1, 8, 1, 64, 65536, 3000, [65536], 3, kv=K)
    np.testing.assert_array_equal(idx[0, 0], np.arange(3000))


# ----------------------------------------------------------------------------- a4 decode
def _decode_case(B, Hq, Hkv, D, L, idx, seq_lens, n_fresh, seed):
    K = synth.kv_cache(seed, synth.STREAM_K, B, Hkv, L, D)
    V = synth.kv_cache(seed, synth.STREAM_V, B, Hkv, L, D)
    _, q = synth.query_trace(seed, B, Hq, 2, D)
    out = asp.sparse_decode(to_dev_bf16(q), to_dev_bf16(K), to_dev_bf16(V),
                            torch.tensor(seq_lens, dtype=torch.int32, device=DEV),
                            torch.from_numpy(idx).to(DEV), n_fresh=n_fresh)
    ref = oracle.sparse_decode(q, K, V, idx, seq_lens, n_fresh)
    return out.cpu().numpy(), ref, (q, K, V)


@pytest.mark.parametrize("G", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("n_fresh", [0, 1, 3])
def test_decode_parity(G, D, n_fresh):
    rng = np.random.default_rng(G * 10 + D + n_fresh)
    B, Hkv, L, k = 2, 2, 1500, 600                      # 600 + n_fresh entries: 3 chunks, ragged
    seq_lens = [1500, 900]
    idx = np.full((B, Hkv, k), -1, np.int32)
    for b in range(B):
        for h in range(Hkv):
            m = min(k - 7, seq_lens[b])
            idx[b, h, :m] = np.sort(rng.choice(seq_lens[b], m, replace=False))
    out, ref, _ = _decode_case(B, Hkv * G, Hkv, D, L, idx, seq_lens, n_fresh, 40 + G)
    assert rel_inf_err(out, ref) <= ATTN_RTOL


@pytest.mark.parametrize("G", [4, 8, 16, 32])
@pytest.mark.parametrize("k,n_fresh", [(128, 1), (256, 1), (300, 0), (383, 1), (384, 0), (384, 1)])
def test_decode_one_item_rows(G, k, n_fresh):
    """Rows of top_k + n_fresh <= 384 entries are ONE decode item of up to 3
    tiles written straight to out (G <= 16); 385 entries and G = 32 take the
    256-entry split + combine.  Every boundary against the oracle, with a
    ragged row and selections that run into the fresh tail."""
    rng = np.random.default_rng(G * 1000 + k + n_fresh)
    B, Hkv, D, L = 2, 2, 128, 1024
    seq_lens = [1024, 333]
    idx = np.full((B, Hkv, k), -1, np.int32)
    for b in range(B):
        for h in range(Hkv):
            m = min(k - 3, seq_lens[b])
            idx[b, h, :m] = np.sort(rng.choice(seq_lens[b], m, replace=False))
    out, ref, _ = _decode_case(B, Hkv * G, Hkv, D, L, idx, seq_lens, n_fresh, 70 + G)
    assert rel_inf_err(out, ref) <= ATTN_RTOL


def test_decode_full_selection_equals_dense():
    """North star: with k = context length, sparse attention == dense."""
    B, Hq, Hkv, D, L = 2, 8, 2, 128, 700
    idx = np.broadcast_to(np.arange(L, dtype=np.int32), (B, Hkv, L)).copy()
    out, ref, (q, K, V) = _decode_case(B, Hq, Hkv, D, L, idx, [L, L], 0, 5)
    dense = oracle.dense_attention(q, K, V, [L, L])
    assert rel_inf_err(out, dense) <= ATTN_RTOL
    assert rel_inf_err(out, ref) <= ATTN_RTOL


def test_decode_edge_cases():
    """Empty set -> 0; one token -> its V row; duplicate fresh tail ignored."""
    B, Hq, Hkv, D, L = 1, 4, 1, 64, 64
    idx = np.full((B, Hkv, 8), -1, np.int32)
    out, _, _ = _decode_case(B, Hq, Hkv, D, L, idx, [L], 0, 9)
    assert np.all(out == 0)
    idx[0, 0, 3] = 17
    out, ref, (_, _, V) = _decode_case(B, Hq, Hkv, D, L, idx, [L], 0, 9)
    np.testing.assert_array_equal(out[0, 0], synth.bf16_bits_to_f32(V[0, 0, 17]))
    idx[0, 0, 4] = 63                                   # also the fresh token
    out, ref, _ = _decode_case(B, Hq, Hkv, D, L, idx, [L], 1, 9)
    assert rel_inf_err(out, ref) <= ATTN_RTOL


# ----------------------------------------------------------------------------- composed step
def _oracle_row_checks(step: DecodeStep, rows, n_fresh=0, lens=None, overlap=None, kv_rows=None):
    """For sampled (b, h): predict / select (band) / decode parity, chained
    (lens: per-batch sequence lengths of a ragged step; default uniform L).
    overlap (a list): also run the UNCHAINED oracle step (oracle q_hat ->
    oracle scores -> oracle top-k) and append each row's Eq. 1 overlap ratio
    |S_gpu & S_oracle| / k.  kv_rows(b, h) ->
    (K, V) bf16 bits [L, D] overrides the plain generator (structured keys)."""
    cfg = step.cfg
    G, D, L, k, W = cfg.group, cfg.head_dim, cfg.seq_len, cfg.top_k, cfg.window
    seed = synth.base_seed(cfg.index)
    qh_g = step.q_hat.cpu().numpy()
    idx_g = step.sel_idx.cpu().numpy()
    out_g = step.out.cpu().numpy()
    bands = 0
    for r in rows:
        b, hl = divmod(int(r), step.n_kv)
        hg = step.h0 + hl
        win, q = synth.query_trace(seed, cfg.batch, cfg.n_q_heads, W, D, b0=b, h0=hg * G,
                                   batch_slice=1, head_slice=G)
        qh_or, _ = oracle.predict(win, step.eps, step.flags)
        assert rel_inf_err(qh_g[b, hl * G:(hl + 1) * G], qh_or[0]) <= Q_HAT_RTOL
        if kv_rows is None:
            K = synth.kv_rows(seed, synth.STREAM_K, b, hg, 0, L, cfg.n_kv_heads, L, D)[None, None]
            V = synth.kv_rows(seed, synth.STREAM_V, b, hg, 0, L, cfg.n_kv_heads, L, D)[None, None]
        else:
            K, V = (x[None, None] for x in kv_rows(b, hg))
        n = L if lens is None else int(lens[b])
        s_or, _ = oracle.score(qh_g[b:b + 1, hl * G:(hl + 1) * G], K, [n])   # chained
        bands += check_selection(idx_g[b, hl], s_or[0, 0], n - n_fresh, k)["band"]
        if overlap is not None:                                              # unchained
            s_un, _ = oracle.score(qh_or, K, [n])
            i_un, _ = oracle.select(s_un, k, [[n]])
            a, c = idx_g[b, hl], i_un[0, 0]
            overlap.append(len(np.intersect1d(a[a >= 0], c[c >= 0])) / max(min(k, n), 1))
        o_or = oracle.sparse_decode(q, K, V, idx_g[b:b + 1, hl:hl + 1], [n], n_fresh)
        assert rel_inf_err(out_g[b, hl * G:(hl + 1) * G], o_or[0]) <= ATTN_RTOL
    return bands


def test_step_tiny_all_rows():
    step = DecodeStep(configs.TINY, DEV)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    _oracle_row_checks(step, range(configs.TINY.batch * configs.TINY.n_kv_heads))


def test_step_qwen3_8b_sampled_rows():
    step = DecodeStep(configs.QWEN3_8B, DEV)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    assert int(step.dev_flags.item()) == 0
    ov = []
    _oracle_row_checks(step, rows_sample(step.cfg.batch * step.n_kv, 32, seed=1), overlap=ov)
    # unchained end to end (oracle q_hat): Eq. 1 overlap >= 0.999
    assert np.mean(ov) >= 0.999 and min(ov) >= 0.99, (np.mean(ov), min(ov))
    del step
    torch.cuda.empty_cache()


def test_step_qwen3_32b_graph_sampled_rows_and_determinism():
    """Config [2] at full size in the launch configuration bench.py times
    (CUDA-graph replay); sampled rows vs the oracle; replays bit-identical."""
    step = DecodeStep(configs.QWEN3_32B, DEV)
    step.fill_synthetic()
    step.capture()
    step.replay()
    torch.cuda.synchronize()
    idx1, out1 = step.sel_idx.clone(), step.out.clone()
    step.replay()
    torch.cuda.synchronize()
    assert torch.equal(idx1, step.sel_idx) and torch.equal(out1, step.out)
    # the deterministic 32-row subset of SURVEY §8(d) / BASELINE.md §3, chained
    # parity on each, and the unchained Eq. 1 overlap ratio
    ov = []
    _oracle_row_checks(step, rows_sample(step.cfg.batch * step.n_kv, 32, seed=2), overlap=ov)
    assert np.mean(ov) >= 0.999 and min(ov) >= 0.99, (np.mean(ov), min(ov))
    del step
    torch.cuda.empty_cache()


def test_step_qwen3_32b_ragged_sampled_rows():
    """Config [2] at full size with bench.py --ragged's length mix (seeded
    uniform in [L/8, L]; the score kernel balances its VALID tiles over the
    SMs): sampled rows -- the shortest and the longest among them -- vs the
    oracle."""
    cfg = configs.QWEN3_32B
    step = DecodeStep(cfg, DEV)
    step.fill_synthetic()
    rng = np.random.default_rng(synth.base_seed(cfg.index) + 99)
    lens = rng.integers(cfg.seq_len // 8, cfg.seq_len + 1, cfg.batch)
    step.seq_lens.copy_(torch.from_numpy(lens.astype(np.int32)))
    step.run()
    torch.cuda.synchronize()
    assert int(step.dev_flags.item()) == 0
    bmin, bmax = int(np.argmin(lens)), int(np.argmax(lens))
    rows = sorted({bmin * step.n_kv, bmax * step.n_kv + 7, *rows_sample(step.cfg.batch * step.n_kv, 4, seed=5)})
    _oracle_row_checks(step, rows, lens=lens)
    del step
    torch.cuda.empty_cache()


def test_layer_packed_step_bit_identical():
    """NEXT-2: one launch per kernel over P_l = 3 stacked layers
    reproduces the three single-layer steps bit for bit, and a packed layer is
    checked against the oracle on sampled rows."""
    cfg = configs.QWEN3_8B.with_(batch=3, seq_len=4096, top_k=256)
    packed = DecodeStep(cfg, DEV, layers=3)
    packed.fill_synthetic()
    packed.run()
    B = cfg.batch
    for layer in range(3):
        one = DecodeStep(cfg, DEV)
        one.fill_synthetic(synth.base_seed(cfg.index) + synth.LAYER_SEED_STRIDE * layer)
        one.run()
        torch.cuda.synchronize()
        rows = slice(layer * B, (layer + 1) * B)
        assert torch.equal(one.q_hat, packed.q_hat[rows])
        assert torch.equal(one.sel_idx, packed.sel_idx[rows])
        assert torch.equal(one.out, packed.out[rows])
    # layer 2 of the pack against the oracle (chained), batch row 1, KV head 5
    sd = synth.base_seed(cfg.index) + 2 * synth.LAYER_SEED_STRIDE
    G, b, h = cfg.group, 1, 5
    K = synth.kv_rows(sd, synth.STREAM_K, b, h, 0, cfg.seq_len, cfg.n_kv_heads, cfg.seq_len,
                      cfg.head_dim)[None, None]
    V = synth.kv_rows(sd, synth.STREAM_V, b, h, 0, cfg.seq_len, cfg.n_kv_heads, cfg.seq_len,
                      cfg.head_dim)[None, None]
    r = 2 * B + b
    qh = packed.q_hat[r:r + 1, h * G:(h + 1) * G].cpu().numpy()
    s_or, _ = oracle.score(qh, K, [cfg.seq_len])
    idx = packed.sel_idx[r:r + 1, h:h + 1].cpu().numpy()
    check_selection(idx[0, 0], s_or[0, 0], cfg.seq_len, cfg.top_k)
    q = from_dev_bf16(packed.q[r:r + 1, h * G:(h + 1) * G])
    o_or = oracle.sparse_decode(q, K, V, idx, [cfg.seq_len])
    assert rel_inf_err(packed.out[r:r + 1, h * G:(h + 1) * G].cpu().numpy(), o_or) <= ATTN_RTOL


def test_kv_head_shards_bit_identical():
    """§8(e): P = 2 KV-head shards reproduce the P = 1 slices bit for bit."""
    cfg = configs.QWEN3_8B.with_(batch=4, seq_len=8192, top_k=512)
    full = DecodeStep(cfg, DEV)
    full.fill_synthetic()
    full.run()
    G = cfg.group
    for r in range(2):
        part = DecodeStep(cfg, DEV, kv_heads=(r * 4, 4))
        part.fill_synthetic()
        part.run()
        torch.cuda.synchronize()
        assert torch.equal(part.sel_idx, full.sel_idx[:, r * 4:(r + 1) * 4])
        assert torch.equal(part.out, full.out[:, r * 4 * G:(r + 1) * 4 * G])
        assert torch.equal(part.q_hat, full.q_hat[:, r * 4 * G:(r + 1) * 4 * G])


def test_step_with_fresh_token():
    cfg = configs.QWEN3_8B.with_(batch=2, seq_len=4096, top_k=256)
    step = DecodeStep(cfg, DEV, n_fresh=1)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    # selection saw all L tokens; decode skips idx in the fresh tail and adds it once
    cfg_rows = rows_sample(cfg.batch * cfg.n_kv_heads, 4, seed=3)
    seed = synth.base_seed(cfg.index)
    out_g = step.out.cpu().numpy()
    idx_g = step.sel_idx.cpu().numpy()
    for r in cfg_rows:
        b, h = divmod(int(r), cfg.n_kv_heads)
        G, D, L = cfg.group, cfg.head_dim, cfg.seq_len
        _, q = synth.query_trace(seed, cfg.batch, cfg.n_q_heads, cfg.window, D, b0=b,
                                 h0=h * G, batch_slice=1, head_slice=G)
        K = synth.kv_rows(seed, synth.STREAM_K, b, h, 0, L, cfg.n_kv_heads, L, D)[None, None]
        V = synth.kv_rows(seed, synth.STREAM_V, b, h, 0, L, cfg.n_kv_heads, L, D)[None, None]
        o_or = oracle.sparse_decode(q, K, V, idx_g[b:b + 1, h:h + 1], [L], 1)
        assert rel_inf_err(out_g[b, h * G:(h + 1) * G], o_or[0]) <= ATTN_RTOL


def test_decode_independent_of_cache_state():
    """Regression: the decode result must not depend on timing (a producer
    WAR race on the token list once showed up only with a cold L2)."""
    cfg = configs.QWEN3_8B.with_(batch=8, seq_len=16384, top_k=1024)
    step = DecodeStep(cfg, DEV)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    ref = step.out.clone()
    junk = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=DEV)
    for it in range(3):
        junk.fill_(it)                                     # evict L2
        asp.sparse_decode(step.q, step.k_cache, step.v_cache, step.seq_lens, step.sel_idx,
                          out=step.out, workspace=step.ws_dec, params=step.p_dec)
        torch.cuda.synchronize()
        assert torch.equal(step.out, ref)


# ----------------------------------------------------------------------------- configs [3], [4]
def test_long_cot_512k_shard_sampled_rows():
    """Config [3] at its longest context (512k tokens, k = 32,768) on the
    per-GPU shard of the 8-GPU run (one KV head): L2-streaming select path,
    32k-entry decode sets; sampled rows vs the oracle."""
    cfg = configs.long_cot(524288)
    step = DecodeStep(cfg, DEV, kv_heads=(5, 1))
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    assert int(step.dev_flags.item()) == 0
    _oracle_row_checks(step, [0, 7])
    del step
    torch.cuda.empty_cache()


@pytest.mark.parametrize("batch", [1, 512])
def test_high_concurrency_sampled_rows(batch):
    """Config [4] end points: Qwen3-8B shape, 4k context, k = 256."""
    cfg = configs.high_concurrency(batch)
    step = DecodeStep(cfg, DEV)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    assert int(step.dev_flags.item()) == 0
    _oracle_row_checks(step, rows_sample(batch * cfg.n_kv_heads, min(6, batch * 8), seed=4))
    del step
    torch.cuda.empty_cache()


# ----------------------------------------------------------------------------- a5 async
def test_async_pipeline_matches_serial():
    """a5: selection for step t+1 on the side stream, overlapped with step
    t's decode and the synthetic forward, gives bit-identical idx and out to
    the same steps run serially on one stream."""
    from paper_2510_07486_b200.pipeline import AsyncPipeline
    cfg = configs.high_concurrency(16).with_(seq_len=8192, top_k=512)
    T = 5
    g = torch.Generator().manual_seed(11)
    B, Hq, Hkv, D = cfg.batch, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
    qts = [torch.randn(B, Hq, D, generator=g).to(DEV) for _ in range(T)]
    qs = [torch.randn(B, Hq, D, generator=g).to(torch.bfloat16).to(DEV) for _ in range(T)]
    kvs = [torch.randn(2, B, Hkv, D, generator=g).to(torch.bfloat16).to(DEV) for _ in range(T)]
    runs = []
    for mode in ("serial", "async"):
        step = DecodeStep(cfg, DEV, n_fresh=1)
        step.fill_synthetic()
        pipe = AsyncPipeline(step, forward_bytes=64 << 20)
        outs, idxs = [], []
        for t in range(T):
            step.q.copy_(qs[t])
            if mode == "async":
                pipe.run_step(qts[t], kvs[t])
            else:
                pipe.run_step_serial(qts[t], kvs[t])
            outs.append(step.out.clone())
            idxs.append(pipe.idx[t % 2].clone())
        pipe.drain()
        torch.cuda.synchronize()
        runs.append((outs, idxs, step))
    (o_s, i_s, _), (o_a, i_a, _) = runs
    for t in range(T):
        assert torch.equal(i_s[t], i_a[t]), t
        assert torch.equal(o_s[t], o_a[t]), t
    # the selections really changed as the window and cache moved
    assert not torch.equal(i_a[0], i_a[T - 1])


# ----------------------------------------------------------------------------- paged pools (NEXT-4)
@pytest.mark.parametrize("G,D,P", [(8, 128, 16), (1, 64, 64), (4, 128, 32), (2, 64, 128),
                                   (2, 64, 16), (16, 128, 32), (32, 64, 16)])
def test_paged_matches_dense_bit_for_bit(G, D, P):
    """The paged entry points return bit for bit what the dense ones return on
    the same logical cache (random page placement, spare pages, ragged
    lengths incl. a row shorter than k and a partial last page, n_fresh = 1),
    and a paged row passes the oracle (chained)."""
    B, Hkv, L, k = 4, 2, 1024, 96
    seed = synth.base_seed(0) + 77 + P
    K = synth.kv_cache(seed, synth.STREAM_K, B, Hkv, L, D)
    V = synth.kv_cache(seed, synth.STREAM_V, B, Hkv, L, D)
    Kd, Vd = to_dev_bf16(K), to_dev_bf16(V)
    lens = [L, 517, 40, 1000]
    sl = torch.tensor(lens, dtype=torch.int32, device=DEV)
    rng = np.random.default_rng(seed)
    qh = torch.from_numpy((rng.standard_normal((B, Hkv * G, D)) * 0.7).astype(np.float32)).to(DEV)
    q = torch.from_numpy(rng.standard_normal((B, Hkv * G, D)).astype(np.float32)).to(DEV).to(torch.bfloat16)
    gen = torch.Generator().manual_seed(seed)
    k_pool, bt = asp.page_pool(Kd, P, gen, spare_pages=5)
    gen = torch.Generator().manual_seed(seed)
    v_pool, bt_v = asp.page_pool(Vd, P, gen, spare_pages=5)
    assert torch.equal(bt, bt_v)
    bt = bt.contiguous()
    s_d = torch.full((B, Hkv, L), np.nan, dtype=torch.float32, device=DEV)
    s_p = torch.full((B, Hkv, L), np.nan, dtype=torch.float32, device=DEV)
    idx_d = asp.score_select(qh, Kd, sl, k, scores=s_d)
    idx_p = asp.score_select_paged(qh, k_pool, bt, sl, k, L, scores=s_p)
    idx_w = asp.score_select_paged(qh, k_pool, bt, sl, k, L)          # workspace path
    torch.cuda.synchronize()
    assert torch.equal(idx_d, idx_p) and torch.equal(idx_p, idx_w)
    for b in range(B):
        assert torch.equal(s_d[b, :, :lens[b]], s_p[b, :, :lens[b]])
    out_d = asp.sparse_decode(q, Kd, Vd, sl, idx_d, n_fresh=1)
    out_p = asp.sparse_decode_paged(q, k_pool, v_pool, bt, sl, idx_p, L, n_fresh=1)
    torch.cuda.synchronize()
    assert torch.equal(out_d, out_p)
    # oracle, chained, on the ragged row b = 1
    b = 1
    so, _ = oracle.score(qh[b:b + 1].cpu().numpy(), K[b:b + 1], [lens[b]])
    for h in range(Hkv):
        check_selection(idx_p[b, h].cpu().numpy(), so[0, h], lens[b], k)
    o_or = oracle.sparse_decode(from_dev_bf16(q[b:b + 1]), K[b:b + 1], V[b:b + 1],
                                idx_p[b:b + 1].cpu().numpy(), [lens[b]], n_fresh=1)
    assert rel_inf_err(out_p[b:b + 1].cpu().numpy(), o_or) <= ATTN_RTOL


# ----------------------------------------------------------------------------- Quest comparator
@pytest.mark.parametrize("G,D,agg", [(8, 128, asp.AGG_MAX), (1, 64, asp.AGG_MAX), (4, 128, asp.AGG_SUM)])
def test_quest_select_parity(G, D, agg):
    """GPU Quest page-bound selection vs the oracle (SPEC page_level_select):
    page sets equal outside the 1e-5 band of the k/P-th bound, every selected
    page expanded to its tokens (ascending, -1 past the length)."""
    B, Hkv, L, P, k = 3, 2, 1000, 16, 128
    seed = synth.base_seed(0) + 313 + G
    K = synth.kv_cache(seed, synth.STREAM_K, B, Hkv, L, D)
    Kd = to_dev_bf16(K)
    lens = [1000, 517, 40]
    sl = torch.tensor(lens, dtype=torch.int32, device=DEV)
    q = (np.random.default_rng(seed).standard_normal((B, Hkv * G, D))).astype(np.float32)
    meta = asp.quest_summarize(Kd, sl, P, k, Hkv * G)
    flags = torch.zeros(1, dtype=torch.int32, device=DEV)
    idx = asp.quest_select(torch.from_numpy(q).to(DEV), meta, Kd, sl, k, P, aggregation=agg,
                           dev_flags=flags).cpu().numpy()
    _, pidx_or, bounds = oracle.quest_select(q, K, lens, k, P, agg)
    for b in range(B):
        npg = (lens[b] + P - 1) // P
        for h in range(Hkv):
            row = idx[b, h]
            pages = row[::P]
            pages = np.where(pages >= 0, pages // P, -1)
            check_selection(pages, bounds[b, h], npg, k // P)
            # expansion: whole pages, ascending, -1 past the length
            exp = np.array([pg * P + e % P if pg >= 0 and pg * P + e % P < lens[b] else -1
                            for e, pg in enumerate(np.repeat(pages, P))])
            np.testing.assert_array_equal(row, exp)
    assert flags.item() & asp.FLAG_SHORT_ROW              # row b = 2 has 3 pages < 8


# ----------------------------------------------------------------------------- a0 append
def test_append_is_exact_data_movement():
    """a0: one kernel writes q_t into the ring slot, bf16(q_t) into
    the current query and the new K / V rows at pos[b] -- bit for bit what
    the equivalent torch copies produce; other state untouched; pos < 0
    skips a row's cache write."""
    cfg = configs.QWEN3_8B.with_(batch=3, seq_len=512, top_k=64)
    step = DecodeStep(cfg, DEV)
    step.fill_synthetic()
    win0, k0, v0 = step.window.clone(), step.k_cache.clone(), step.v_cache.clone()
    g = torch.Generator(device="cpu").manual_seed(5)
    q_t = torch.randn(3, 32, 128, generator=g).to(DEV)
    k_new = torch.randn(3, 8, 128, generator=g).to(torch.bfloat16).to(DEV)
    v_new = torch.randn(3, 8, 128, generator=g).to(torch.bfloat16).to(DEV)
    pos = torch.tensor([511, 7, -1], dtype=torch.int32, device=DEV)
    slot = step.ring_start
    step.append(q_t, k_new, v_new, pos)
    torch.cuda.synchronize()
    ref_w = win0.clone()
    ref_w[:, :, slot] = q_t
    assert torch.equal(step.window, ref_w)
    assert torch.equal(step.q, q_t.to(torch.bfloat16))
    ref_k, ref_v = k0.clone(), v0.clone()
    ref_k[0, :, 511], ref_k[1, :, 7] = k_new[0], k_new[1]
    ref_v[0, :, 511], ref_v[1, :, 7] = v_new[0], v_new[1]
    assert torch.equal(step.k_cache, ref_k) and torch.equal(step.v_cache, ref_v)
    assert step.ring_start == (slot + 1) % cfg.window


# ----------------------------------------------------------------------------- NEXT-1 gather / dual rank
def test_gather_filtered_bit_equal():
    """SPEC gather_filtered: packed rows bit-equal to the cache
    rows, zeros for -1 / out-of-length entries; all indices -> the cache."""
    cfg = configs.QWEN3_8B.with_(batch=2, seq_len=512, top_k=64)
    step = DecodeStep(cfg, DEV)
    step.fill_synthetic()
    step.seq_lens.copy_(torch.tensor([512, 300], dtype=torch.int32))
    step.run()
    idx = step.sel_idx.clone()
    idx[0, 0, 5] = -1
    idx[1, 2, 7] = 400                                     # >= seq_lens[1]
    io = torch.empty_like(idx)
    ko, vo = asp.gather_filtered(step.k_cache, step.v_cache, step.seq_lens, idx, n_fresh=1,
                                 idx_out=io)
    torch.cuda.synchronize()
    for b in range(2):
        n = int(step.seq_lens[b])
        for h in range(8):
            exp_i = [j if 0 <= int(idx[b, h, j]) < n - 1 else -1 for j in range(64)]
            assert io[b, h].tolist() == exp_i
    for b in range(2):
        for h in range(8):
            for j in range(64):
                t = int(idx[b, h, j])
                ok = 0 <= t < int(step.seq_lens[b])
                exp_k = step.k_cache[b, h, t] if ok else torch.zeros_like(ko[b, h, j])
                exp_v = step.v_cache[b, h, t] if ok else torch.zeros_like(vo[b, h, j])
                assert torch.equal(ko[b, h, j], exp_k) and torch.equal(vo[b, h, j], exp_v)
    full = torch.arange(512, dtype=torch.int32, device=DEV).expand(2, 8, 512).contiguous()
    step.seq_lens.fill_(512)
    ka, va = asp.gather_filtered(step.k_cache, step.v_cache, step.seq_lens, full)
    assert torch.equal(ka, step.k_cache) and torch.equal(va, step.v_cache)


def _dual_rank(tmp_path, *args):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "dual.npz")
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "disagg_two_rank.py"), out,
                        *args], capture_output=True, text=True, timeout=240, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return dict(np.load(out))


def _dual_rank_oracle_check(d):
    """Each Inference-Rank output against the oracle: attention of the step's
    query over the rows of the selection it used (global indices, the
    Cache Rank's) plus its own fresh token at L - 1 (n_fresh = 1, R12)."""
    cfg = configs.QWEN3_8B.with_(batch=2, seq_len=1024, top_k=128)
    seed = synth.base_seed(cfg.index)
    L = cfg.seq_len
    K = synth.kv_cache(seed, synth.STREAM_K, cfg.batch, cfg.n_kv_heads, L, cfg.head_dim)
    V = synth.kv_cache(seed, synth.STREAM_V, cfg.batch, cfg.n_kv_heads, L, cfg.head_dim)
    for t in range(len(d["outs"])):
        K[:, :, L - 1] = d["kvs"][t][0]
        V[:, :, L - 1] = d["kvs"][t][1]
        q_bits = synth.f32_to_bf16_bits(d["q_ts"][t])
        sel = d["sent"][int(d["used"][t])]
        o_or = oracle.sparse_decode(q_bits, K, V, sel, [L] * cfg.batch, n_fresh=1)
        assert rel_inf_err(d["outs"][t], o_or) <= ATTN_RTOL, t


def test_dual_rank_disaggregation_matches_single_rank_and_oracle(tmp_path):
    """NEXT-1: an Inference Rank and a Cache Rank (two processes on
    one GPU, gloo with host staging; one process group per direction) with the
    'wait' stall policy: step t uses selection t, the outputs are bit for bit
    the single-rank a5 pipeline's on the same inputs, and each matches the
    oracle over the selection it used plus the fresh token."""
    d = _dual_rank(tmp_path, "--reference", "--steps", "4")
    assert d["used"].tolist() == [0, 1, 2, 3]
    np.testing.assert_array_equal(d["outs"], d["ref_outs"])
    _dual_rank_oracle_check(d)


def test_dual_rank_late_cache_rank_reuses_previous_selection(tmp_path):
    """SPEC S:590 stall policy 'reuse': the Cache Rank sends sel(2) half a
    second late; the Inference Rank does not wait -- step 2 attends with
    sel(1) (plus its fresh token) and takes the newest selection as soon as it
    has arrived.  Every step's output matches the oracle over the selection it
    actually used."""
    d = _dual_rank(tmp_path, "--policy", "reuse", "--late", "1", "--steps", "5")
    used = d["used"].tolist()
    # step t can use at most sel(t); sel(2) is half a second late, so step 2
    # attends with an older one; selections are taken in order, newest first
    assert used[0] == 0 and all(u <= t for t, u in enumerate(used)), used
    assert used[2] <= 1, used
    assert all(b >= a for a, b in zip(used, used[1:])) and used[-1] >= 2, used
    _dual_rank_oracle_check(d)


def test_predict_bf16_window():
    """NEXT-3: a bf16 query ring (ASP_WINDOW_BF16) -- q_hat bit-identical to
    the fp32 path on the exactly widened values, and within the north-star
    tolerance of the oracle; unsupported combinations are refused."""
    for flags in (0, asp.ASSEMBLY_SINGLE, asp.SIGN_NEGATED, asp.DOUBLE_SOFTMAX,
                  asp.ASSEMBLY_SINGLE | asp.NORM_NONE):
        for B, Hq, W, D in ((3, 5, 16, 128), (2, 4, 9, 64), (1, 3, 2, 128)):
            win, _ = synth.query_trace(synth.base_seed(1) + W, B, Hq, W, D)
            wb = torch.from_numpy(win).to(DEV).to(torch.bfloat16)
            wf = wb.float()
            ring = W // 3
            g_b = asp.predict_query(wb, flags=flags, ring_start=ring)
            g_f = asp.predict_query(wf, flags=flags, ring_start=ring)
            assert torch.equal(g_b, g_f), (flags, W)
            ref, cond = oracle.predict(wf.cpu().numpy(), 1e-2, flags, ring)
            assert cond == 0
            assert rel_inf_err(g_b.cpu().numpy(), ref) <= Q_HAT_RTOL
    w32 = torch.zeros(1, 2, 32, 64, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(asp.AsyncSpadeError):
        asp.predict_query(w32)
    w8 = torch.zeros(1, 2, 8, 64, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(asp.AsyncSpadeError):
        asp.predict_query(w8, flags=asp.ASSEMBLY_PER_WINDOW)


def test_bf16_window_step_and_append():
    """A bf16 query ring end to end: asyncspade_append rounds q_t into the
    slot, the step predicts from it exactly as from the widened fp32 ring."""
    cfg = configs.QWEN3_8B.with_(batch=2, seq_len=1024, top_k=128)
    sb = DecodeStep(cfg, DEV, window_dtype=torch.bfloat16)
    sb.fill_synthetic()
    q_t = torch.randn(2, 32, 128, generator=torch.Generator().manual_seed(9)).to(DEV)
    slot = sb.ring_start
    sb.append(q_t)
    torch.cuda.synchronize()
    assert torch.equal(sb.window[:, :, slot], q_t.to(torch.bfloat16))
    sf = DecodeStep(cfg, DEV)
    sf.fill_synthetic()
    sf.window.copy_(sb.window.float())
    sf.q.copy_(sb.q)
    sf.ring_start, sf.p_pred.ring_start = sb.ring_start, sb.ring_start
    sb.run()
    sf.run()
    torch.cuda.synchronize()
    assert torch.equal(sb.q_hat, sf.q_hat)
    assert torch.equal(sb.sel_idx, sf.sel_idx) and torch.equal(sb.out, sf.out)


def test_step_group16_sampled_rows():
    """NEXT-3: GQA group of 16 (e.g. 128 query / 8 KV heads) through the whole
    step -- score (5 TMEM accumulator stages), select, decode (32-row P
    operand) -- against the oracle on sampled rows."""
    cfg = configs.Config("g16", 0, 2, 32, 2, 128, 4096, 256, 16)
    step = DecodeStep(cfg, DEV)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    assert int(step.dev_flags.item()) == 0
    _oracle_row_checks(step, range(cfg.batch * cfg.n_kv_heads))


def test_step_mqa_group32_sampled_rows():
    """NEXT-3: multi-query attention -- 32 query heads on ONE KV head (G = 32:
    score N = 96 with 2 TMEM accumulator stages and a 5-stage K ring, decode
    with a 64-row P operand and 256 TMEM columns) -- against the oracle."""
    cfg = configs.Config("mqa32", 0, 3, 32, 1, 128, 4096, 256, 16)
    step = DecodeStep(cfg, DEV, n_fresh=1)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    assert int(step.dev_flags.item()) == 0
    _oracle_row_checks(step, range(cfg.batch * cfg.n_kv_heads), n_fresh=1)


@pytest.mark.parametrize("G", [16, 32])
def test_score_select_large_groups_multi_tile_ranges(G):
    """G = 16 / 32 with several 128-token tiles per persistent CTA (the MMA
    issuer groups tiles; G = 32 has only 2 TMEM accumulator stages): band-rule
    parity on every row against the oracle."""
    B, Hkv, D, L, k = 2, 1, 128, 32768, 2048
    lens = [L, 20000]
    idx, _, s_or, flags = _score_select_case(B, Hkv * G, Hkv, D, L, k, lens, seed=400 + G)
    for b in range(B):
        check_selection(idx[b, 0], s_or[b, 0], lens[b], k)


@pytest.mark.parametrize("G", [16, 32])
def test_step_large_groups_multi_item(G):
    """G = 16 / 32 through the whole step with several decode work items and
    score tiles per persistent CTA (the pipelined slot / phase paths), sampled
    rows against the oracle."""
    cfg = configs.Config(f"g{G}_multi", 0, 4, 8 * G, 8, 128, 8192, 2048, 16)
    step = DecodeStep(cfg, DEV)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    assert int(step.dev_flags.item()) == 0
    _oracle_row_checks(step, rows_sample(cfg.batch * cfg.n_kv_heads, 4, seed=G))
    del step
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", [configs.QWEN3_8B.with_(batch=3, seq_len=4096, top_k=700),
                                 configs.QWEN3_8B.with_(batch=3, seq_len=4096, top_k=256),
                                 configs.Config("mqa64", 0, 3, 64, 1, 128, 4096, 700, 16)],
                         ids=["split-k", "one-item", "mqa64-virtual-heads"])
def test_decode_head_major_out(cfg):
    """ABI 2: the split-K combine (and a one-item row's direct write, and the
    MQA virtual-head split) writes `out` through (row, head) strides;
    head-major [Hq, B, D] holds bit for bit the dense result transposed, so
    KV-head shards concatenate."""
    step = DecodeStep(cfg, DEV, n_fresh=1)
    step.fill_synthetic()
    step.run()
    torch.cuda.synchronize()
    dense = step.out.clone()
    p_hm = asp.decode_params(step.q, step.k_cache, step.v_cache, cfg.top_k, 1, out_head_major=True)
    for _ in range(2):
        hm = asp.sparse_decode(step.q, step.k_cache, step.v_cache, step.seq_lens, step.sel_idx,
                               params=p_hm)
        torch.cuda.synchronize()
        assert hm.shape == (cfg.n_q_heads, cfg.batch, cfg.head_dim)
        assert torch.equal(hm.transpose(0, 1), dense)


def test_head_major_shards_concatenate_to_the_full_output():
    """§8(e): with head-major outputs ([Hq/P, B, D] per KV-head shard) the
    shards' outputs concatenated along the head axis are bit for bit the
    unsharded run's [B, Hq, D] output transposed -- the all-gather is a plain
    concatenation (shard.gather_heads)."""
    cfg = configs.QWEN3_8B.with_(batch=3, seq_len=4096, top_k=256)
    full = DecodeStep(cfg, DEV, n_fresh=1)
    full.fill_synthetic()
    full.run()
    parts = []
    for r in range(4):
        part = DecodeStep(cfg, DEV, kv_heads=(2 * r, 2), n_fresh=1, out_head_major=True)
        part.fill_synthetic()
        part.run()
        parts.append(part.out)
    torch.cuda.synchronize()
    cat = torch.cat(parts, dim=0)                     # what all_gather_into_tensor produces
    assert cat.shape == (cfg.n_q_heads, cfg.batch, cfg.head_dim)
    assert torch.equal(cat.transpose(0, 1), full.out)

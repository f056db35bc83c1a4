"""Pins for the CPU oracle (oracle/asp_oracle.c) -- checks it against what the
paper and mathematics fix, never against itself: closed forms, special cases,
invariants, brute force and independent library routines (numpy).  Each test
names the passage / SURVEY §8(c) reading it pins.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2510_07486_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MODES = [oracle.ASSEMBLY_MASKED_SHARED, oracle.ASSEMBLY_SINGLE, oracle.ASSEMBLY_PER_WINDOW,
         oracle.ASSEMBLY_MASKED_SHARED | oracle.DOUBLE_SOFTMAX]


def _softmax(v):
    v = np.asarray(v, np.float64)
    e = np.exp(v - v.max())
    return e / e.sum()


# ----------------------------------------------------------------------------- predict
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("W", [2, 4, 16])
def test_constant_window_is_exact(mode, W):
    """a constant window predicts the constant, bit-exactly
    (every candidate is a convex combination of identical vectors)."""
    rng = np.random.default_rng(1)
    q = rng.standard_normal(64).astype(np.float32)
    win = np.broadcast_to(q, (3, W, 64)).copy()
    qh, cond = oracle.predict(win, 1e-2, mode)
    assert cond == 0
    assert np.array_equal(qh, np.broadcast_to(q, (3, 64)))


@pytest.mark.parametrize("mode", MODES)
def test_w2_returns_newest(mode):
    """W = 2 leaves one usable weight, so q_hat = Q_t in
    every mode (masked-shared == per-window at W = 2)."""
    rng = np.random.default_rng(2)
    win = rng.standard_normal((5, 2, 32)).astype(np.float32)
    qh, _ = oracle.predict(win, 1e-2, mode)
    assert np.array_equal(qh, win[:, 1])


def test_w1_passthrough():
    """S:208 warm-up rule: fewer than two queries -> passthrough."""
    win = np.random.default_rng(3).standard_normal((2, 1, 16)).astype(np.float32)
    qh, _ = oracle.predict(win)
    assert np.array_equal(qh, win[:, 0])


def test_large_eps_closed_form_masked_shared():
    """Readings R3-R6 pinned by a closed form: with eps -> infinity the ridge
    weights vanish, every row softmax is uniform over its n_j = min(j, W-1)
    entries, so q_hat = (1/W) sum_j mean(Q[W-n_j..W-1]).  (NOT the window
    mean that S:202 claims -- it differs.)"""
    rng = np.random.default_rng(4)
    W, D = 8, 48
    win = rng.standard_normal((6, W, D)).astype(np.float32)
    qh, _ = oracle.predict(win, 1e12, oracle.ASSEMBLY_MASKED_SHARED)
    Q = win.astype(np.float64)
    n = W - 1
    exp = np.zeros((6, D))
    for j in range(1, W + 1):
        nj = min(j, n)
        exp += Q[:, W - nj:].mean(axis=1)
    exp /= W
    np.testing.assert_allclose(qh, exp, rtol=0, atol=1e-6)
    assert np.abs(exp - Q.mean(axis=1)).max() > 1e-2   # S:202's "window mean" is wrong


def test_large_eps_closed_form_single_and_per_window():
    """Eq. 4 with uniform weights: mean(Q[1..W-1]); Eq. 5 literal
    (m = W-1): (1/n) sum_k mean(Q[W-k..W-1])."""
    rng = np.random.default_rng(5)
    W, D = 6, 40
    win = rng.standard_normal((4, W, D)).astype(np.float32)
    Q = win.astype(np.float64)
    qs, _ = oracle.predict(win, 1e12, oracle.ASSEMBLY_SINGLE)
    np.testing.assert_allclose(qs, Q[:, 1:].mean(axis=1), atol=1e-6, rtol=0)
    qp, _ = oracle.predict(win, 1e12, oracle.ASSEMBLY_PER_WINDOW)
    n = W - 1
    exp = sum(Q[:, W - k:].mean(axis=1) for k in range(1, n + 1)) / n
    np.testing.assert_allclose(qp, exp, atol=1e-6, rtol=0)


def _orthonormal_window(W, D, a):
    """History rows Q[0..n-1] = e_1..e_n, newest Q[W-1] = sum a_i e_i."""
    n = W - 1
    win = np.zeros((W, D), np.float32)
    for i in range(n):
        win[i, i] = 1.0
    win[W - 1, :n] = a
    return win


@pytest.mark.parametrize("negated", [False, True])
def test_orthonormal_history_closed_form(negated):
    """Alg. 1 Step 3 pinned exactly: G0 = I, mean diag = 1, so with
    relative eps = 1e-2 the ridge weights are omega = a / 1.01 (generalises
    S:164).  Then every assembly mode has a closed-form softmax mixture."""
    W, D = 5, 16
    n = W - 1
    a = np.array([0.5, -1.0, 2.0, 0.25], np.float32)
    win = _orthonormal_window(W, D, a)
    Q = win.astype(np.float64)
    om = a.astype(np.float64) / 1.01
    s = -1.0 if negated else 1.0
    flag = oracle.SIGN_NEGATED if negated else 0
    # masked-shared (R4/R5/R6)
    exp = np.zeros(D)
    for j in range(1, W + 1):
        nj = min(j, n)
        r = _softmax(s * om[:nj])
        exp += r @ Q[W - nj:]
    exp /= W
    qh, _ = oracle.predict(win[None], 1e-2, oracle.ASSEMBLY_MASKED_SHARED | flag)
    np.testing.assert_allclose(qh[0], exp, atol=1e-7, rtol=0)
    # single (Eq. 4)
    qs, _ = oracle.predict(win[None], 1e-2, oracle.ASSEMBLY_SINGLE | flag)
    np.testing.assert_allclose(qs[0], _softmax(s * om) @ Q[1:], atol=1e-7, rtol=0)
    # double softmax (literal Step 4)
    p = _softmax(s * om)
    exp2 = sum(_softmax(p[:min(j, n)]) @ Q[W - min(j, n):] for j in range(1, W + 1)) / W
    qd, _ = oracle.predict(win[None], 1e-2,
                           oracle.ASSEMBLY_MASKED_SHARED | oracle.DOUBLE_SOFTMAX | flag)
    np.testing.assert_allclose(qd[0], exp2, atol=1e-7, rtol=0)
    # per-window (Eq. 5): H_k = e_{n-k+1}..e_n -> omega_k = a[n-k:] / 1.01
    exp3 = sum(_softmax(s * a[n - k:].astype(np.float64) / 1.01) @ Q[W - k:]
               for k in range(1, n + 1)) / n
    qp, _ = oracle.predict(win[None], 1e-2, oracle.ASSEMBLY_PER_WINDOW | flag)
    np.testing.assert_allclose(qp[0], exp3, atol=1e-7, rtol=0)


def test_sign_example_from_spec():
    """softmax([ln 2, 0]) = [2/3, 1/3]; negated -> [1/3, 2/3].
    Realised through SINGLE mode at W = 3 with absolute eps chosen so the
    ridge weights are exactly [ln 2, 0] on an orthonormal history."""
    ln2 = np.log(2.0)
    win = np.zeros((3, 8), np.float32)
    win[0, 0] = 1.0
    win[1, 1] = 1.0
    # omega = a / (1 + eps): pick a0 = ln2 * (1 + eps) in fp32 exactly enough
    eps = 2.0 ** -20
    win[2, 0] = np.float32(ln2 * (1 + eps))
    qs, _ = oracle.predict(win[None], eps, oracle.ASSEMBLY_SINGLE | oracle.EPS_ABSOLUTE)
    # weights (2/3, 1/3) applied to Q[1], Q[2]
    exp = (2 / 3) * win[1].astype(np.float64) + (1 / 3) * win[2].astype(np.float64)
    np.testing.assert_allclose(qs[0], exp, atol=2e-7)
    qn, _ = oracle.predict(win[None], eps,
                           oracle.ASSEMBLY_SINGLE | oracle.EPS_ABSOLUTE | oracle.SIGN_NEGATED)
    exp = (1 / 3) * win[1].astype(np.float64) + (2 / 3) * win[2].astype(np.float64)
    np.testing.assert_allclose(qn[0], exp, atol=2e-7)


@pytest.mark.parametrize("mode", MODES)
def test_power_of_two_scale_equivariance(mode):
    """S:199, S:307 scale equivariance; with relative eps a 2^k scaling is
    exact in floating point, so q_hat scales bit-exactly."""
    rng = np.random.default_rng(6)
    win = rng.standard_normal((8, 16, 128)).astype(np.float32)
    q1, _ = oracle.predict(win, 1e-2, mode)
    q8, _ = oracle.predict(win * np.float32(8.0), 1e-2, mode)
    assert np.array_equal(q8, q1 * np.float32(8.0))


def test_raw_single_window_reproduces_exact_linear_recurrence():
    """North star: 'the regressor reproduces exactly-linear query sequences'
    (reading R17: the raw, NORM_NONE single-window ridge regression).  With an
    exact order-(W-1) recurrence Q_s = sum_i c_i Q_{s-i} over dyadic c_i and
    small-integer starts (exact in fp32), Eq. 4's shifted weights predict the
    next element of the recurrence."""
    rng = np.random.default_rng(7)
    for trial in range(20):
        W, D = 5, 64
        n = W - 1
        c = rng.choice([-0.5, -0.25, 0.25, 0.5, 0.125], size=n)
        seq = [rng.integers(-3, 4, D).astype(np.float64) for _ in range(n)]
        for _ in range(2):
            seq.append(sum(c[i] * seq[-1 - i] for i in range(n)))
        win = np.array(seq[:W], np.float32)
        assert np.array_equal(win.astype(np.float64), np.array(seq[:W]))  # exact in fp32
        qh, cond = oracle.predict(win[None], 1e-12,
                                  oracle.ASSEMBLY_SINGLE | oracle.NORM_NONE | oracle.EPS_ABSOLUTE)
        assert cond == 0
        np.testing.assert_allclose(qh[0], seq[W], atol=1e-9 * (1 + np.abs(seq[W]).max()))


@pytest.mark.parametrize("mode", [oracle.ASSEMBLY_MASKED_SHARED, oracle.ASSEMBLY_SINGLE,
                                  oracle.ASSEMBLY_PER_WINDOW])
def test_convexity(mode):
    """S:143 / S:221: softmax modes output a convex combination of window
    queries: ||q_hat|| <= max_p ||Q_p||."""
    rng = np.random.default_rng(8)
    win = rng.standard_normal((64, 16, 64)).astype(np.float32) * rng.uniform(
        0.1, 10, (64, 16, 1)).astype(np.float32)
    qh, _ = oracle.predict(win, 1e-2, mode)
    assert np.all(np.linalg.norm(qh, axis=1)
                  <= np.linalg.norm(win, axis=2).max(axis=1) * (1 + 1e-6))


def test_ridge_solve_matches_numpy_linalg():
    """Alg. 1 Step 3 via an independent library solve: numpy.linalg.solve of
    (G0 + eps I) omega = beta, then the SINGLE-mode softmax mixture."""
    for W in (4, 9, 16):
        win = synth.query_trace(123 + W, 4, 2, W, 128)[0].reshape(8, W, 128)
        qs, _ = oracle.predict(win, 1e-2, oracle.ASSEMBLY_SINGLE)
        for r in range(8):
            Q = win[r].astype(np.float64)
            H, y = Q[:-1], Q[-1]
            G0 = H @ H.T
            om = np.linalg.solve(G0 + 1e-2 * np.mean(np.diag(G0)) * np.eye(W - 1), H @ y)
            np.testing.assert_allclose(qs[r], _softmax(om) @ Q[1:], rtol=0,
                                       atol=1e-6 * np.abs(Q).max())


def test_not_pd_and_nonfinite_passthrough():
    """S:69 not-PD error class and S:208 passthrough: a negative absolute eps
    on a zero history has a non-positive pivot -> flag 2, q_hat = newest; a
    NaN window -> flag 1, passthrough."""
    win = np.zeros((1, 4, 8), np.float32)
    win[0, 3] = np.arange(8)
    qh, cond = oracle.predict(win, -1.0, oracle.EPS_ABSOLUTE)
    assert cond & oracle.FLAG_NOT_PD and np.array_equal(qh[0], win[0, 3])
    win2 = np.ones((1, 4, 8), np.float32)
    win2[0, 1, 2] = np.nan
    qh2, cond2 = oracle.predict(win2)
    assert cond2 & oracle.FLAG_NONFINITE and np.array_equal(qh2[0], win2[0, 3])


def test_ring_start_rotation():
    """Ring mapping (§8(b)): logical slot j lives at physical (ring_start+j)%W."""
    rng = np.random.default_rng(10)
    win = rng.standard_normal((3, 7, 32)).astype(np.float32)
    q0, _ = oracle.predict(win)
    rot = np.roll(win, 3, axis=1)        # physical[(3 + j) % W] = logical[j]
    q3, _ = oracle.predict(rot, ring_start=3)
    assert np.array_equal(q0, q3)


# ----------------------------------------------------------------------------- score
def _kv(rng, B, H, L, D):
    return synth.f32_to_bf16_bits(rng.standard_normal((B, H, L, D)).astype(np.float32))


def test_score_basis_query_reads_first_column():
    """q_hat = e_1 -> score of token n = K[n, 0]."""
    rng = np.random.default_rng(11)
    K = _kv(rng, 2, 2, 50, 64)
    q = np.zeros((2, 4, 64), np.float32)
    q[..., 0] = 1.0
    s, _ = oracle.score(q, K, 50)
    np.testing.assert_array_equal(s, synth.bf16_bits_to_f32(K[..., 0]).astype(np.float64))


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_score_matches_numpy_matmul(G):
    """Alg. 1 Step 7 with a library fp64 matmul per head, reduced
    over the group by elementwise max (R10) or sum."""
    rng = np.random.default_rng(12 + G)
    B, Hkv, L, D = 2, 2, 97, 128
    K = _kv(rng, B, Hkv, L, D)
    q = rng.standard_normal((B, Hkv * G, D)).astype(np.float32)
    s, _ = oracle.score(q, K, [97, 60])
    s_sum, _ = oracle.score(q, K, [97, 60], oracle.AGG_SUM)
    Kf = synth.bf16_bits_to_f32(K).astype(np.float64)
    for b in range(B):
        for h in range(Hkv):
            per = Kf[b, h] @ q[b, h * G:(h + 1) * G].astype(np.float64).T   # [L, G]
            ln = [97, 60][b]
            np.testing.assert_allclose(s[b, h, :ln], per.max(axis=1)[:ln], rtol=1e-13, atol=1e-12)
            np.testing.assert_allclose(s_sum[b, h, :ln], per.sum(axis=1)[:ln], rtol=1e-13,
                                       atol=1e-12)
            assert np.all(np.isneginf(s[b, h, ln:]))


# ----------------------------------------------------------------------------- select
def _brute_topk(s, k):
    """Brute force: full lexicographic sort by (-score, index)."""
    order = np.lexsort((np.arange(len(s)), -s))
    return np.sort(order[:k])


def test_select_matches_brute_force_with_ties():
    """S:93, S:710 'top-k matches a brute-force full sort', with the north
    star's lower-index tie-break (R9) -- scores drawn from a 16-value codebook
    so exact ties are everywhere."""
    rng = np.random.default_rng(13)
    for L, k in [(1000, 100), (257, 32), (4096, 256), (64, 64)]:
        s = rng.integers(0, 16, (6, L)).astype(np.float64) * 0.37
        idx, cond = oracle.select(s, k)
        for r in range(6):
            np.testing.assert_array_equal(idx[r], _brute_topk(s[r], k))
        s2 = rng.standard_normal((6, L))
        idx2, _ = oracle.select(s2, k)
        for r in range(6):
            np.testing.assert_array_equal(idx2[r], _brute_topk(s2[r], k))


def test_select_special_cases():
    """S:282-283 and R9/R13: k = L -> identity; increasing -> last k; all
    equal -> first k; positive scaling invariant; short rows padded."""
    L = 300
    ident, _ = oracle.select(np.random.default_rng(14).standard_normal(L), L)
    np.testing.assert_array_equal(ident, np.arange(L))
    inc, _ = oracle.select(np.arange(L, dtype=np.float64), 7)
    np.testing.assert_array_equal(inc, np.arange(L - 7, L))
    eq, _ = oracle.select(np.full(L, 3.5), 9)
    np.testing.assert_array_equal(eq, np.arange(9))
    s = np.random.default_rng(15).standard_normal(L)
    np.testing.assert_array_equal(oracle.select(s, 20)[0], oracle.select(s * 7.25, 20)[0])
    short, cond = oracle.select(np.arange(10, dtype=np.float64)[None], 16, [10])
    assert cond & oracle.FLAG_SHORT_ROW
    np.testing.assert_array_equal(short[0], list(range(10)) + [-1] * 6)


def test_select_nan_sorts_last():
    """R14: NaN scores rank below every number."""
    s = np.array([1.0, np.nan, 0.5, -3.0, np.nan])
    idx, cond = oracle.select(s, 3)
    assert cond & oracle.FLAG_NONFINITE
    np.testing.assert_array_equal(idx, [0, 2, 3])


def test_select_spec_golden_examples():
    """tests/golden/spec_select_examples.json: SPEC S:91-92 examples, the
    tie case restated under the north-star tie-break (lower index wins)."""
    with open(os.path.join(GOLDEN, "spec_select_examples.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        idx, _ = oracle.select(np.array(c["scores"], np.float64), c["k"])
        assert idx.tolist() == c["expect"], c


# ----------------------------------------------------------------------------- decode
def _attn_numpy(q, K, V, toks, scale):
    """Library evaluation of softmax attention (fp64 numpy)."""
    l = (K[toks] @ q) * scale
    p = np.exp(l - l.max())
    return (p / p.sum()) @ V[toks]


def test_decode_matches_numpy_and_dense_at_full_selection():
    """North star / S:310: with k = L (every token), sparse attention
    equals dense attention; both equal a numpy fp64 evaluation."""
    rng = np.random.default_rng(16)
    B, Hq, Hkv, L, D = 2, 4, 2, 90, 64
    K, V = _kv(rng, B, Hkv, L, D), _kv(rng, B, Hkv, L, D)
    q = synth.f32_to_bf16_bits(rng.standard_normal((B, Hq, D)).astype(np.float32))
    idx = np.broadcast_to(np.arange(L, dtype=np.int32), (B, Hkv, L)).copy()
    out = oracle.sparse_decode(q, K, V, idx, L)
    dense = oracle.dense_attention(q, K, V, L)
    np.testing.assert_array_equal(out, dense)
    Kf, Vf, qf = (synth.bf16_bits_to_f32(x).astype(np.float64) for x in (K, V, q))
    for b in range(B):
        for hq in range(Hq):
            h = hq // (Hq // Hkv)
            ref = _attn_numpy(qf[b, hq], Kf[b, h], Vf[b, h], np.arange(L), 1 / np.sqrt(D))
            np.testing.assert_allclose(out[b, hq], ref, rtol=1e-6, atol=1e-7)


def test_decode_special_cases():
    """one token -> V0; equal logits (q = 0) -> mean V; a single
    index -> that V; idx order and -1 padding do not matter; the n_fresh tail
    is attended once even if also selected (R12)."""
    rng = np.random.default_rng(17)
    B, Hq, Hkv, L, D = 1, 2, 1, 40, 64
    K, V = _kv(rng, B, Hkv, L, D), _kv(rng, B, Hkv, L, D)
    Vf = synth.bf16_bits_to_f32(V).astype(np.float64)
    q = synth.f32_to_bf16_bits(rng.standard_normal((B, Hq, D)).astype(np.float32))
    one = oracle.sparse_decode(q, K, V, np.array([[[-1, 5, -1]]], np.int32), L)
    np.testing.assert_array_equal(one[0, 0], Vf[0, 0, 5].astype(np.float32))
    zq = np.zeros_like(q)
    mean = oracle.sparse_decode(zq, K, V, np.array([[[1, 3, 7, 8]]], np.int32), L)
    np.testing.assert_allclose(mean[0, 1], Vf[0, 0, [1, 3, 7, 8]].mean(axis=0), rtol=1e-6,
                               atol=1e-7)
    a = oracle.sparse_decode(q, K, V, np.array([[[2, 9, 30, -1]]], np.int32), L, n_fresh=1)
    b = oracle.sparse_decode(q, K, V, np.array([[[30, -1, 9, 2]]], np.int32), L, n_fresh=1)
    c = oracle.sparse_decode(q, K, V, np.array([[[30, 39, 9, 2]]], np.int32), L, n_fresh=1)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a, c)
    Kf, qf = synth.bf16_bits_to_f32(K).astype(np.float64), synth.bf16_bits_to_f32(q)
    ref = _attn_numpy(qf[0, 0].astype(np.float64), Kf[0, 0], Vf[0, 0], [2, 9, 30, 39],
                      1 / np.sqrt(D))
    np.testing.assert_allclose(a[0, 0], ref, rtol=1e-6, atol=1e-7)


# ----------------------------------------------------------------------------- generator
def test_generator_determinism_and_sharding():
    """§8(e): inputs are a pure function of the global index, so a shard
    equals the matching slice of the whole tensor; two draws are identical."""
    s = synth.base_seed(0)
    full = synth.kv_cache(s, synth.STREAM_K, 2, 4, 33, 16)
    part = synth.kv_cache(s, synth.STREAM_K, 2, 4, 33, 16, b0=1, h0=2, batch_slice=1,
                          head_slice=2)
    np.testing.assert_array_equal(full[1:2, 2:4], part)
    w1, q1 = synth.query_trace(s, 2, 8, 16, 32)
    w2, q2 = synth.query_trace(s, 2, 8, 16, 32, h0=4, head_slice=4)
    np.testing.assert_array_equal(w1[:, 4:], w2)
    np.testing.assert_array_equal(q1[:, 4:], q2)
    x = synth.bf16_bits_to_f32(synth.kv_cache(s, synth.STREAM_V, 4, 8, 512, 128))
    assert abs(float(x.mean())) < 0.01 and abs(float(x.std()) - 1.0) < 0.01


# ----------------------------------------------------------------------------- Quest comparator
def _quest_case(seed, B=2, Hq=4, Hkv=2, D=16, L=64):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, Hq, D)).astype(np.float32)
    K = synth.kv_cache(seed, synth.STREAM_K, B, Hkv, L, D)
    return q, K


def test_quest_page_size_one_is_token_topk():
    """SPEC S:395 example 1: P = 1 -> the page bound is the exact dot product
    and the selection equals token-level top-k."""
    q, K = _quest_case(3)
    lens = [64, 37]
    idx, _, bounds = oracle.quest_select(q, K, lens, 8, 1)
    s, _ = oracle.score(q, K, lens)
    np.testing.assert_array_equal(bounds[:, :, :37], s[:, :, :37])
    ref, _ = oracle.select(s, 8, np.repeat(lens, 2).reshape(2, 2))
    np.testing.assert_array_equal(idx, ref)


def test_quest_bound_brute_force_and_upper_bound_property():
    """every token's true score is <= its page's bound
    (checked exhaustively over every token of every page), and the C bound
    matches an independent numpy min / max reduction of the decoded keys."""
    q, K = _quest_case(5, L=80)
    P = 16
    lens = [80, 70]
    bounds, _ = oracle.page_bounds(q, K, lens, P)
    s, _ = oracle.score(q, K, lens)
    kv = K.astype(np.uint32) << 16
    kf = kv.view(np.float32).astype(np.float64)
    for b in range(2):
        for h in range(2):
            for j in range((lens[b] + P - 1) // P):
                t0, t1 = j * P, min(lens[b], (j + 1) * P)
                assert np.all(s[b, h, t0:t1] <= bounds[b, h, j] + 1e-12)
                mx, mn = kf[b, h, t0:t1].max(0), kf[b, h, t0:t1].min(0)
                qg = q[b, 2 * h:2 * h + 2].astype(np.float64)
                u = np.maximum(qg * mx, qg * mn).sum(1).max()
                assert abs(u - bounds[b, h, j]) <= 1e-12 * max(1.0, abs(u))
            assert np.all(np.isneginf(bounds[b, h, (lens[b] + P - 1) // P:]))


def test_quest_constant_pages_select_whole_token_pages():
    """SPEC S:396 example 2: keys identical within every page -> the bound is
    the exact token score, and the selected pages are the pages of the
    token-level selection (page-aligned budget)."""
    rng = np.random.default_rng(11)
    B, Hq, Hkv, D, L, P = 1, 2, 1, 8, 64, 8
    per_page = rng.standard_normal((B, Hkv, L // P, D)).astype(np.float32)
    Kf = np.repeat(per_page, P, axis=2)
    K = (Kf.view(np.uint32) >> 16).astype(np.uint16)            # exact bf16 truncation
    q = rng.standard_normal((B, Hq, D)).astype(np.float32)
    idx, pidx, bounds = oracle.quest_select(q, K, [L], 16, P)
    s, _ = oracle.score(q, K, [L])
    np.testing.assert_allclose(bounds[0, 0], s[0, 0, ::P], rtol=0, atol=0)
    tok, _ = oracle.select(s, 16)
    assert set(tok[0, 0] // P) == set(pidx[0, 0])
    np.testing.assert_array_equal(np.sort(idx[0, 0]), np.sort(
        np.concatenate([np.arange(pg * P, pg * P + P) for pg in sorted(pidx[0, 0])])))


def test_quest_short_rows_and_partial_last_page():
    """Tokens past the length are -1; fewer pages than the budget pad -1."""
    q, K = _quest_case(9, B=1, Hkv=1, Hq=1, L=64)
    idx, pidx, _ = oracle.quest_select(q, K, [20], 48, 16)     # 2 pages exist, 3 wanted
    assert list(pidx[0, 0]) == [0, 1, -1]
    np.testing.assert_array_equal(idx[0, 0], np.r_[np.arange(20), -np.ones(28, int)])


def test_select_signed_zero_ties_and_nan_fill():
    """R14 + R9, pinned independently of the oracle's own code: -0.0 and +0.0
    are EQUAL numbers (IEEE 754 5.11), so they tie and the lower index wins
    whichever sign it carries; NaNs rank below every number and fill a row
    that has fewer than k numbers in index order (the brute-force
    lexicographic sort with NaN mapped below -inf)."""
    cases = [
        (np.array([-1.0, -0.0, 0.0, -0.0, 2.0]), 3, [1, 2, 4]),
        (np.array([0.0, -0.0]), 1, [0]),
        (np.array([-0.0, 0.0]), 1, [0]),
        (np.array([-0.0, -5.0, 0.0, 0.0]), 2, [0, 2]),
        (np.array([np.nan, 1.0, np.nan, np.nan]), 3, [0, 1, 2]),
        (np.array([np.nan, -np.inf, np.nan]), 2, [0, 1]),
    ]
    for s, k, exp in cases:
        idx, cond = oracle.select(s, k)
        np.testing.assert_array_equal(idx, exp)
        assert bool(cond & oracle.FLAG_NONFINITE) == bool(np.isnan(s).any())
        key = np.where(np.isnan(s), -np.inf, s)          # brute force, NaN below everything
        order = np.lexsort((np.arange(len(s)), np.isnan(s), -key))
        np.testing.assert_array_equal(np.sort(order[:k]), exp)
    # a random row salted with signed zeros and NaNs against the brute force
    rng = np.random.default_rng(41)
    s = rng.integers(-3, 4, 500).astype(np.float64)
    s[rng.random(500) < 0.3] = -0.0
    s[rng.random(500) < 0.05] = np.nan
    idx, _ = oracle.select(s, 300)
    key = np.where(np.isnan(s), -np.inf, s)
    order = np.lexsort((np.arange(500), np.isnan(s), -key))
    np.testing.assert_array_equal(idx, np.sort(order[:300]))


def test_ar1_prediction_beats_random_selection():
    """SPEC S:712-713 sanity check (SURVEY §8(c) 'end-to-end sanity'): on
    SPEC's AR(1) query traces (alpha 0.95) the selection made with the
    predicted query q_hat overlaps the selection of the TRUE next query
    q_{t+1} (Eq. 1) at least 3x as much as a random selection
    (k/N = 1/8).  Keys ~ N(0,1), N = 2048, k = 256, W = 16."""
    rng = np.random.default_rng(2025)
    B, Hq, W, D, N, k = 4, 8, 16, 64, 2048, 256
    T = W + 1
    q = np.empty((B, Hq, T, D))
    q[:, :, 0] = rng.standard_normal((B, Hq, D))
    for t in range(1, T):
        q[:, :, t] = 0.95 * q[:, :, t - 1] + 0.05 * rng.standard_normal((B, Hq, D))
    win = q[:, :, :W].astype(np.float32)
    nxt = q[:, :, W].astype(np.float32)
    K = synth.f32_to_bf16_bits(rng.standard_normal((B, Hq, N, D)).astype(np.float32))
    qh, cond = oracle.predict(win)
    assert cond == 0
    s_hat, _ = oracle.score(qh, K, [N] * B)
    s_true, _ = oracle.score(nxt, K, [N] * B)
    i_hat, _ = oracle.select(s_hat, k)
    i_true, _ = oracle.select(s_true, k)
    ov = np.mean([len(np.intersect1d(i_hat[b, h], i_true[b, h])) / k
                  for b in range(B) for h in range(Hq)])
    assert ov >= 3 * k / N, ov
    # and a random index set really sits near k / N (the baseline is meaningful)
    rnd = np.mean([len(np.intersect1d(np.sort(rng.choice(N, k, replace=False)), i_true[b, h])) / k
                   for b in range(B) for h in range(Hq)])
    assert abs(rnd - k / N) < 0.03, rnd


def test_decode_values_narrower_than_keys_absorbed_mla():
    """NEXT-3 absorbed MLA: the value of a token is the first Dv
    dims of its key row (the latent); the oracle's decode over V narrower than
    K equals numpy softmax attention with logits over all D key dims and the
    weighted sum over the Dv value dims."""
    rng = np.random.default_rng(57)
    B, Hq, Hkv, D, Dv, L = 2, 4, 1, 96, 64, 40
    q = synth.f32_to_bf16_bits(rng.standard_normal((B, Hq, D)).astype(np.float32))
    K = synth.f32_to_bf16_bits(rng.standard_normal((B, Hkv, L, D)).astype(np.float32))
    V = np.ascontiguousarray(K[..., :Dv])
    idx = np.stack([np.stack([np.sort(rng.choice(L - 1, 9, replace=False))]) for _ in range(B)]).astype(np.int32)
    out = oracle.sparse_decode(q, K, V, idx, [L] * B, n_fresh=1, sm_scale=0.11)
    assert out.shape == (B, Hq, Dv)
    for b in range(B):
        toks = list(idx[b, 0]) + [L - 1]
        Kf = synth.bf16_bits_to_f32(K[b, 0]).astype(np.float64)
        for hq in range(Hq):
            qf = synth.bf16_bits_to_f32(q[b, hq]).astype(np.float64)
            l = 0.11 * (Kf[toks] @ qf)
            p = np.exp(l - l.max())
            p /= p.sum()
            ref = p @ Kf[toks, :Dv]
            np.testing.assert_allclose(out[b, hq], ref, rtol=1e-6, atol=1e-7)

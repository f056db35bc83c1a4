"""Helpers for GPU-vs-oracle parity tests (tolerances from BASELINE.json's
north star, defined precisely in DESIGN.md §5)."""
from __future__ import annotations

import numpy as np

Q_HAT_RTOL = 1e-4      # max_(b,hq) ||q_gpu - q_or||_inf / ||q_or||_inf
SCORE_BAND = 1e-5      # index sets exact outside +-1e-5 relative of the k-th score
ATTN_RTOL = 2e-3       # max_(b,hq) ||o_gpu - o_or||_inf / ||o_or||_inf


def rel_inf_err(gpu: np.ndarray, ref: np.ndarray) -> float:
    """max over leading rows of ||gpu - ref||_inf / ||ref||_inf (last axis)."""
    g = gpu.reshape(-1, gpu.shape[-1]).astype(np.float64)
    r = ref.reshape(-1, ref.shape[-1]).astype(np.float64)
    num = np.abs(g - r).max(axis=1)
    den = np.maximum(np.abs(r).max(axis=1), 1e-30)
    return float((num / den).max())


def check_selection(idx_gpu: np.ndarray, scores_or: np.ndarray, length: int, k: int) -> dict:
    """Band rule for one row: the GPU set (ascending, -1 padded) must equal
    the oracle's outside +-SCORE_BAND*|s*| of the oracle's k-th score s*.
    Returns stats; raises AssertionError on violation."""
    idx = np.asarray(idx_gpu)
    if length <= k:
        exp = np.concatenate([np.arange(length), -np.ones(k - length, np.int64)])
        assert np.array_equal(idx, exp), "short row must hold every token then -1"
        return {"band": 0}
    assert np.all(np.diff(idx) > 0), "indices must be strictly ascending"
    assert idx[0] >= 0 and idx[-1] < length, "index out of range"
    s = np.asarray(scores_or[:length], np.float64)
    s_k = np.sort(s)[::-1][k - 1]
    tau = SCORE_BAND * max(abs(s_k), 1e-30)
    sel = np.zeros(length, bool)
    sel[idx] = True
    must = s > s_k + tau
    never = s < s_k - tau
    assert np.all(sel[must]), f"missed {int((must & ~sel).sum())} tokens above the band"
    assert not np.any(sel[never]), f"took {int((never & sel).sum())} tokens below the band"
    return {"band": int((~must & ~never).sum())}


def rows_sample(n_rows: int, n: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    n = min(n, n_rows)
    pick = set([0, n_rows - 1])
    while len(pick) < n:
        pick.add(int(rng.integers(0, n_rows)))
    return np.array(sorted(pick))

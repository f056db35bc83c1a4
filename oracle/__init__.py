"""CPU oracle for the AsyncSpade decode hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2510_07486_b200``) never imports it; it shares no code
with the CUDA path.  The arithmetic lives in ``asp_oracle.c`` (plain C99,
fp64, one thread); this module only marshals numpy arrays through ctypes.

Each wrapper names the paper passage its C function follows (``P:<line>`` =
line of reference/PAPER.md).  Pins: tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "asp_oracle.c")
_LIB = os.path.join(_HERE, "libasp_oracle.so")

# condition bits (documented convention shared with the ABI by value only)
FLAG_NONFINITE = 1
FLAG_NOT_PD = 2
FLAG_SHORT_ROW = 4

ASSEMBLY_MASKED_SHARED = 0
ASSEMBLY_SINGLE = 1
ASSEMBLY_PER_WINDOW = 2
SIGN_NEGATED = 1 << 4
EPS_ABSOLUTE = 1 << 5
NORM_NONE = 1 << 6
DOUBLE_SOFTMAX = 1 << 7

AGG_MAX = 0
AGG_SUM = 1


def build(force: bool = False) -> str:
    """Compile asp_oracle.c into libasp_oracle.so (gcc, IEEE fp: no fast-math,
    no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-ffp-contract=off",
             "-fno-fast-math", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i32, u32, f64, vp = ctypes.c_int32, ctypes.c_uint32, ctypes.c_double, ctypes.c_void_p
        lib.asp_oracle_predict.argtypes = [i32, i32, i32, i32, f64, u32, vp, vp]
        lib.asp_oracle_predict.restype = u32
        lib.asp_oracle_score.argtypes = [i32, i32, i32, i32, i32, vp, vp, vp, i32, vp]
        lib.asp_oracle_score.restype = u32
        lib.asp_oracle_page_bounds.argtypes = [i32, i32, i32, i32, i32, i32, vp, vp, vp, i32, vp]
        lib.asp_oracle_page_bounds.restype = u32
        lib.asp_oracle_select.argtypes = [i32, i32, vp, vp, i32, vp]
        lib.asp_oracle_select.restype = u32
        lib.asp_oracle_sparse_decode.argtypes = [i32, i32, i32, i32, i32, i32, i32, f64,
                                                 vp, vp, vp, vp, vp, vp]
        lib.asp_oracle_sparse_decode.restype = u32
        lib.asp_oracle_dense_attention.argtypes = [i32, i32, i32, i32, i32, f64,
                                                   vp, vp, vp, vp, vp]
        lib.asp_oracle_dense_attention.restype = u32
        _lib = lib
    return _lib


def _c(a: np.ndarray, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def predict(q_window: np.ndarray, eps: float = 1e-2, flags: int = 0, ring_start: int = 0):
    """a1: next-query prediction (Eq. 4-5; Alg. 1 Steps 1-6,
    P:497-524).  q_window: fp32 [..., W, D] (any leading dims).
    Returns (q_hat fp32 [..., D], condition bits)."""
    w = _c(q_window, np.float32)
    *lead, W, D = w.shape
    rows = int(np.prod(lead)) if lead else 1
    out = np.empty((rows, D), np.float32)
    cond = _load().asp_oracle_predict(rows, W, D, ring_start, float(eps), flags, _p(w), _p(out))
    return out.reshape(*lead, D), int(cond)


def score(q_hat: np.ndarray, k_cache: np.ndarray, seq_lens, agg: int = AGG_MAX):
    """a2: criticality scores (Alg. 1 Step 7; GQA P:260).
    q_hat fp32 [B, Hq, D]; k_cache bf16 bits uint16 [B, Hkv, L, D].
    Returns (fp64 scores [B, Hkv, L] with -inf past seq_len, bits)."""
    q = _c(q_hat, np.float32)
    k = _c(k_cache, np.uint16)
    B, Hq, D = q.shape
    _, Hkv, L, D2 = k.shape
    assert D == D2 and Hq % Hkv == 0
    sl = _c(np.broadcast_to(np.asarray(seq_lens), (B,)), np.int32)
    out = np.empty((B, Hkv, L), np.float64)
    cond = _load().asp_oracle_score(B, Hq, Hkv, D, L, _p(sl), _p(q), _p(k), agg, _p(out))
    return out, int(cond)


def select(scores: np.ndarray, top_k: int, row_lens=None):
    """a3: per-row top-k, lower index wins ties, ascending, -1 padded
    (readings R9, R13, R14).  scores [..., L] (cast to fp64).
    Returns (int32 [..., top_k], bits)."""
    s = _c(scores, np.float64)
    *lead, L = s.shape
    rows = int(np.prod(lead)) if lead else 1
    if row_lens is None:
        rl = np.full(rows, L, np.int32)
    else:
        rl = _c(np.broadcast_to(np.asarray(row_lens), tuple(lead)).reshape(rows), np.int32)
    out = np.empty((rows, top_k), np.int32)
    cond = _load().asp_oracle_select(rows, L, _p(rl), _p(s), top_k, _p(out))
    return out.reshape(*lead, top_k), int(cond)


def sparse_decode(q: np.ndarray, k_cache: np.ndarray, v_cache: np.ndarray, sel_idx: np.ndarray,
                  seq_lens, n_fresh: int = 0, sm_scale: float | None = None):
    """a4: attention over the selected tokens U the n_fresh tail (P:190,
    P:266; reading R12).  q bf16 bits [B, Hq, D]; caches bf16 bits
    [B, Hkv, L, D]; sel_idx int32 [B, Hkv, k].  Returns fp32 [B, Hq, D]."""
    qq = _c(q, np.uint16)
    k = _c(k_cache, np.uint16)
    v = _c(v_cache, np.uint16)
    ix = _c(sel_idx, np.int32)
    B, Hq, D = qq.shape
    _, Hkv, L, _ = k.shape
    Dv = v.shape[-1]
    if Dv < D:
        # values narrower than the keys (absorbed MLA: the latent is
        # the first Dv key dims): zero-extended to D -- marshalling only, the
        # extra output columns are sum_j p_j * 0 and are dropped
        v = np.ascontiguousarray(np.concatenate(
            [v, np.zeros(v.shape[:-1] + (D - Dv,), np.uint16)], axis=-1))
    top_k = ix.shape[-1]
    if sm_scale is None:
        sm_scale = 1.0 / np.sqrt(D)
    sl = _c(np.broadcast_to(np.asarray(seq_lens), (B,)), np.int32)
    out = np.empty((B, Hq, D), np.float32)
    _load().asp_oracle_sparse_decode(B, Hq, Hkv, D, L, top_k, n_fresh, float(sm_scale),
                                     _p(sl), _p(qq), _p(k), _p(v), _p(ix), _p(out))
    return np.ascontiguousarray(out[..., :Dv])


def dense_attention(q: np.ndarray, k_cache: np.ndarray, v_cache: np.ndarray, seq_lens,
                    sm_scale: float | None = None):
    """Dense attention over all tokens -- what sparse_decode
    must equal when the selection is every token."""
    qq = _c(q, np.uint16)
    k = _c(k_cache, np.uint16)
    v = _c(v_cache, np.uint16)
    B, Hq, D = qq.shape
    _, Hkv, L, _ = k.shape
    if sm_scale is None:
        sm_scale = 1.0 / np.sqrt(D)
    sl = _c(np.broadcast_to(np.asarray(seq_lens), (B,)), np.int32)
    out = np.empty((B, Hq, D), np.float32)
    _load().asp_oracle_dense_attention(B, Hq, Hkv, D, L, float(sm_scale), _p(sl), _p(qq),
                                       _p(k), _p(v), _p(out))
    return out


def page_bounds(q: np.ndarray, k_cache: np.ndarray, seq_lens, page_size: int, agg: int = AGG_MAX):
    """Quest comparator: per-page upper bounds of q . k (SPEC page_level_select,
    S:392-400; the paper's Quest baseline P:356).  q fp32 [B, Hq, D]; k_cache
    bf16 bits [B, Hkv, L, D].  Returns (fp64 [B, Hkv, ceil(L / P)], bits)."""
    qq = _c(q, np.float32)
    k = _c(k_cache, np.uint16)
    B, Hq, D = qq.shape
    _, Hkv, L, _ = k.shape
    NP = (L + page_size - 1) // page_size
    sl = _c(np.broadcast_to(np.asarray(seq_lens), (B,)), np.int32)
    out = np.empty((B, Hkv, NP), np.float64)
    cond = _load().asp_oracle_page_bounds(B, Hq, Hkv, D, L, page_size, _p(sl), _p(qq), _p(k),
                                          agg, _p(out))
    return out, int(cond)


def quest_select(q: np.ndarray, k_cache: np.ndarray, seq_lens, top_k: int, page_size: int,
                 agg: int = AGG_MAX):
    """Quest comparator, SPEC page_level_select: the top_k /
    page_size pages with the largest bound (ties to the lower page, the
    token selector's rule) and all their tokens, ascending; positions past
    the row's length and missing pages are -1.  Returns (idx int32
    [B, Hkv, top_k], page idx, bounds)."""
    B = q.shape[0]
    Hkv = k_cache.shape[1]
    bounds, _ = page_bounds(q, k_cache, seq_lens, page_size, agg)
    lens = np.broadcast_to(np.asarray(seq_lens), (B,))
    n_pages = (lens + page_size - 1) // page_size
    pidx, _ = select(bounds, top_k // page_size, np.repeat(n_pages, Hkv).reshape(B, Hkv))
    idx = np.full((B, Hkv, top_k), -1, np.int32)
    for b in range(B):
        for h in range(Hkv):
            for e in range(top_k):
                pg = pidx[b, h, e // page_size]
                t = pg * page_size + e % page_size if pg >= 0 else -1
                idx[b, h, e] = t if t < lens[b] else -1
    return idx, pidx, bounds


def step(q_window, q, k_cache, v_cache, seq_lens, top_k, eps=1e-2, flags=0, n_fresh=0,
         ring_start=0, agg=AGG_MAX):
    """c1 -> c2 -> c3 -> c4 composed: one decode step."""
    B, Hq, W, D = q_window.shape
    Hkv = k_cache.shape[1]
    q_hat, _ = predict(q_window, eps, flags, ring_start)
    s, _ = score(q_hat, k_cache, seq_lens, agg)
    rl = np.repeat(np.broadcast_to(np.asarray(seq_lens), (B,)), Hkv).reshape(B, Hkv)
    idx, _ = select(s, top_k, rl)
    out = sparse_decode(q, k_cache, v_cache, idx, seq_lens, n_fresh)
    return q_hat, s, idx, out

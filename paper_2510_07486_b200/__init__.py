"""paper_2510_07486_b200 -- B200-native AsyncSpade decode hot path.

Thin Python binding of the C ABI in include/asyncspade.h (libasyncspade.so,
sm_100a).  Functions keep the ABI's names and only marshal arguments: every
step of the path runs in the library's CUDA kernels.  torch provides device
memory and streams; nothing here computes.  There is no CPU fallback: if the
library or a CUDA device is missing, calls raise.

    predict_query   a1  q_hat from the query window           (Alg.1 Steps 1-6)
    score_select    a2+a3  q_hat.K scores + per-row top-k
    sparse_decode   a4  attention over the selected K/V
    score_select_paged / sparse_decode_paged   the same over a paged KV pool
                        (block table, HND pages)
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libasyncspade.so")

ABI_VERSION = 2
ASP_OK = 0
FLAG_NONFINITE, FLAG_NOT_PD, FLAG_SHORT_ROW = 1, 2, 4
ASSEMBLY_MASKED_SHARED, ASSEMBLY_SINGLE, ASSEMBLY_PER_WINDOW = 0, 1, 2
SIGN_NEGATED, EPS_ABSOLUTE, NORM_NONE, DOUBLE_SOFTMAX = 1 << 4, 1 << 5, 1 << 6, 1 << 7
WINDOW_BF16 = 1 << 8
AGG_MAX, AGG_SUM = 0, 1

EXPORTED_SYMBOLS = (
    "asyncspade_append", "asyncspade_predict_query", "asyncspade_score_select_workspace", "asyncspade_score_select",
    "asyncspade_sparse_decode_workspace", "asyncspade_sparse_decode",
    "asyncspade_score_select_paged", "asyncspade_sparse_decode_paged",
    "asyncspade_gather_filtered",
    "asyncspade_quest_meta_bytes", "asyncspade_quest_summarize",
    "asyncspade_quest_select_workspace", "asyncspade_quest_select",
    "asyncspade_status_string", "asyncspade_abi_version",
)


class PredictParams(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("n_q_heads", ctypes.c_int32),
                ("window", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("ring_start", ctypes.c_int32), ("eps", ctypes.c_float),
                ("flags", ctypes.c_uint32)]


class SelectParams(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("n_q_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("top_k", ctypes.c_int32), ("max_seq_len", ctypes.c_int32),
                ("aggregation", ctypes.c_int32),
                ("k_stride_b", ctypes.c_int64), ("k_stride_h", ctypes.c_int64),
                ("k_stride_t", ctypes.c_int64)]


class DecodeParams(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("n_q_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("top_k", ctypes.c_int32), ("n_fresh", ctypes.c_int32),
                ("max_seq_len", ctypes.c_int32), ("sm_scale", ctypes.c_float),
                ("k_stride_b", ctypes.c_int64), ("k_stride_h", ctypes.c_int64),
                ("k_stride_t", ctypes.c_int64), ("v_stride_b", ctypes.c_int64),
                ("v_stride_h", ctypes.c_int64), ("v_stride_t", ctypes.c_int64),
                ("out_stride_b", ctypes.c_int64), ("out_stride_h", ctypes.c_int64),
                ("v_head_dim", ctypes.c_int32)]


class AppendParams(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("n_q_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("window", ctypes.c_int32), ("ring_slot", ctypes.c_int32),
                ("max_seq_len", ctypes.c_int32),
                ("k_stride_b", ctypes.c_int64), ("k_stride_h", ctypes.c_int64),
                ("k_stride_t", ctypes.c_int64), ("v_stride_b", ctypes.c_int64),
                ("v_stride_h", ctypes.c_int64), ("v_stride_t", ctypes.c_int64),
                ("window_bf16", ctypes.c_int32)]


class PagedKV(ctypes.Structure):
    _fields_ = [("page_size", ctypes.c_int32), ("max_pages_per_seq", ctypes.c_int32),
                ("num_pages", ctypes.c_int32)]


class AsyncSpadeError(RuntimeError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    """Load libasyncspade.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        # ASYNCSPADE_LIB selects an instrumented build of the same library
        # (scripts/, development only); the default is the in-tree product.
        path = os.environ.get("ASYNCSPADE_LIB", LIB_PATH)
        if not os.path.exists(path):
            raise AsyncSpadeError(
                f"{path} missing: run `python -m paper_2510_07486_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        vp, sz = ctypes.c_void_p, ctypes.c_size_t
        L.asyncspade_append.argtypes = [ctypes.POINTER(AppendParams), vp, vp, vp, vp, vp, vp, vp,
                                        vp, vp]
        L.asyncspade_append.restype = ctypes.c_int32
        L.asyncspade_gather_filtered.argtypes = [ctypes.POINTER(DecodeParams), vp, vp, vp, vp, vp,
                                                 vp, vp, vp]
        L.asyncspade_gather_filtered.restype = ctypes.c_int32
        L.asyncspade_predict_query.argtypes = [ctypes.POINTER(PredictParams), vp, vp, vp, vp]
        L.asyncspade_predict_query.restype = ctypes.c_int32
        L.asyncspade_score_select_workspace.argtypes = [ctypes.POINTER(SelectParams)]
        L.asyncspade_score_select_workspace.restype = sz
        L.asyncspade_score_select.argtypes = [ctypes.POINTER(SelectParams), vp, vp, vp, vp, vp,
                                              vp, sz, vp, vp]
        L.asyncspade_score_select.restype = ctypes.c_int32
        L.asyncspade_sparse_decode_workspace.argtypes = [ctypes.POINTER(DecodeParams)]
        L.asyncspade_sparse_decode_workspace.restype = sz
        L.asyncspade_sparse_decode.argtypes = [ctypes.POINTER(DecodeParams), vp, vp, vp, vp, vp,
                                               vp, vp, sz, vp]
        L.asyncspade_sparse_decode.restype = ctypes.c_int32
        L.asyncspade_score_select_paged.argtypes = [ctypes.POINTER(SelectParams),
                                                    ctypes.POINTER(PagedKV), vp, vp, vp, vp, vp,
                                                    vp, vp, sz, vp, vp]
        L.asyncspade_score_select_paged.restype = ctypes.c_int32
        L.asyncspade_sparse_decode_paged.argtypes = [ctypes.POINTER(DecodeParams),
                                                     ctypes.POINTER(PagedKV), vp, vp, vp, vp, vp,
                                                     vp, vp, vp, sz, vp]
        L.asyncspade_sparse_decode_paged.restype = ctypes.c_int32
        L.asyncspade_quest_meta_bytes.argtypes = [ctypes.POINTER(SelectParams), ctypes.c_int32]
        L.asyncspade_quest_meta_bytes.restype = sz
        L.asyncspade_quest_summarize.argtypes = [ctypes.POINTER(SelectParams), ctypes.c_int32,
                                                 vp, vp, vp, vp]
        L.asyncspade_quest_summarize.restype = ctypes.c_int32
        L.asyncspade_quest_select_workspace.argtypes = [ctypes.POINTER(SelectParams),
                                                        ctypes.c_int32]
        L.asyncspade_quest_select_workspace.restype = sz
        L.asyncspade_quest_select.argtypes = [ctypes.POINTER(SelectParams), ctypes.c_int32, vp, vp,
                                              vp, vp, vp, sz, vp, vp]
        L.asyncspade_quest_select.restype = ctypes.c_int32
        L.asyncspade_status_string.argtypes = [ctypes.c_int32]
        L.asyncspade_status_string.restype = ctypes.c_char_p
        L.asyncspade_abi_version.argtypes = []
        L.asyncspade_abi_version.restype = ctypes.c_int32
        if L.asyncspade_abi_version() != ABI_VERSION:
            raise AsyncSpadeError("libasyncspade ABI version mismatch")
        _lib = L
    return _lib


def status_string(code: int) -> str:
    return lib().asyncspade_status_string(code).decode()


def _check(code: int, what: str) -> None:
    if code != ASP_OK:
        raise AsyncSpadeError(f"{what}: {status_string(code)} ({code})")


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _u16(t: torch.Tensor) -> torch.Tensor:
    """bf16 tensors are passed as their raw bit pattern."""
    return t if t.dtype != torch.bfloat16 else t.view(torch.int16)


# --------------------------------------------------------------------------- params
def predict_params(q_window: torch.Tensor, eps=1e-2, flags=0, ring_start=0) -> PredictParams:
    B, Hq, W, D = q_window.shape
    if q_window.dtype == torch.bfloat16:
        flags |= WINDOW_BF16                 # a bf16 ring (ASP_WINDOW_BF16)
    return PredictParams(B, Hq, W, D, ring_start, eps, flags)


def select_params(q_hat: torch.Tensor, k_cache: torch.Tensor, top_k: int,
                  aggregation: int = AGG_MAX) -> SelectParams:
    B, Hq, D = q_hat.shape
    _, Hkv, L, _ = k_cache.shape
    sb, sh, st, sd = k_cache.stride()
    if sd != 1:
        raise AsyncSpadeError("k_cache must have unit stride along head_dim")
    return SelectParams(B, Hq, Hkv, D, top_k, L, aggregation, sb, sh, st)


def decode_params(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, top_k: int,
                  n_fresh: int = 0, sm_scale: float | None = None,
                  out_head_major: bool = False, v_head_dim: int = 0) -> DecodeParams:
    """out_head_major: `out` is [Hq, B, Dv] (a KV-head shard's block of the
    gathered [Hq_total, B, Dv] output) instead of [B, Hq, Dv].  v_head_dim:
    the value width (0: head_dim); absorbed MLA passes v_cache = k_cache and
    the latent width 512 < head_dim 576."""
    B, Hq, D = q.shape
    _, Hkv, L, _ = k_cache.shape
    if k_cache.stride(3) != 1 or v_cache.stride(3) != 1:
        raise AsyncSpadeError("caches must have unit stride along head_dim")
    if sm_scale is None:
        sm_scale = D ** -0.5
    dv = v_head_dim or D
    osb, osh = (dv, B * dv) if out_head_major else (0, 0)
    return DecodeParams(B, Hq, Hkv, D, top_k, n_fresh, L, sm_scale, *k_cache.stride()[:3],
                        *v_cache.stride()[:3], osb, osh, v_head_dim)


def score_select_workspace(p: SelectParams) -> int:
    return int(lib().asyncspade_score_select_workspace(ctypes.byref(p)))


def sparse_decode_workspace(p: DecodeParams) -> int:
    return int(lib().asyncspade_sparse_decode_workspace(ctypes.byref(p)))


def _workspace(nbytes: int, device) -> torch.Tensor:
    """A workspace for any entry point: zero-filled once (the decode call's
    arrival counters must start at zero; every call leaves them at zero)."""
    return torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)


# NVTX ranges per entry point (SURVEY §5 profiling), on when ASP_NVTX=1: ncu
# --nvtx / nsys timelines then show each call; off by default (host-side cost).
_NVTX = os.environ.get("ASP_NVTX", "0") == "1"


def _nvtx(fn):
    if not _NVTX:
        return fn
    import functools

    @functools.wraps(fn)
    def wrapped(*a, **kw):
        torch.cuda.nvtx.range_push(fn.__name__)
        try:
            return fn(*a, **kw)
        finally:
            torch.cuda.nvtx.range_pop()
    return wrapped


# --------------------------------------------------------------------------- entry points
@_nvtx
def append(q_t: torch.Tensor, q_window: torch.Tensor | None, ring_slot: int, *,
           q_cur: torch.Tensor | None = None, k_new: torch.Tensor | None = None,
           v_new: torch.Tensor | None = None, k_cache: torch.Tensor | None = None,
           v_cache: torch.Tensor | None = None, pos: torch.Tensor | None = None,
           stream=None) -> None:
    """a0 -> asyncspade_append: q_t fp32 [B, Hq, D] into window slot
    `ring_slot` (q_window may be None), bf16(q_t) into q_cur, k_new / v_new
    [B, Hkv, D] into the caches at pos[b]."""
    if q_window is not None:
        B, Hq, W, D = q_window.shape
    else:
        (B, Hq, D), W, ring_slot = q_t.shape, 1, 0
    kc = k_cache if k_cache is not None else v_cache
    Hkv = kc.shape[1] if kc is not None else 1
    L = kc.shape[2] if kc is not None else 1
    ks = k_cache.stride()[:3] if k_cache is not None else (0, 0, 0)
    vs = v_cache.stride()[:3] if v_cache is not None else (0, 0, 0)
    p = AppendParams(B, Hq, Hkv, D, W, ring_slot, L, *ks, *vs,
                     1 if q_window is not None and q_window.dtype == torch.bfloat16 else 0)
    _check(lib().asyncspade_append(ctypes.byref(p), _ptr(q_t),
                                   _ptr(_u16(q_window) if q_window is not None else None),
                                   _ptr(_u16(q_cur) if q_cur is not None else None),
                                   _ptr(_u16(k_new) if k_new is not None else None),
                                   _ptr(_u16(v_new) if v_new is not None else None),
                                   _ptr(_u16(k_cache) if k_cache is not None else None),
                                   _ptr(_u16(v_cache) if v_cache is not None else None),
                                   _ptr(pos), _stream(stream)),
           "asyncspade_append")


@_nvtx
def predict_query(q_window: torch.Tensor, q_hat: torch.Tensor | None = None, *, eps: float = 1e-2,
                  flags: int = 0, ring_start: int = 0, dev_flags: torch.Tensor | None = None,
                  stream=None, params: PredictParams | None = None) -> torch.Tensor:
    """a1 -> asyncspade_predict_query.  q_window fp32 or bf16 [B, Hq, W, D] (ring
    order per ring_start); returns q_hat fp32 [B, Hq, D]."""
    p = params or predict_params(q_window, eps, flags, ring_start)
    if q_hat is None:
        q_hat = torch.empty(q_window.shape[0], q_window.shape[1], q_window.shape[3],
                            dtype=torch.float32, device=q_window.device)
    _check(lib().asyncspade_predict_query(ctypes.byref(p), _ptr(_u16(q_window)), _ptr(q_hat),
                                          _ptr(dev_flags), _stream(stream)),
           "asyncspade_predict_query")
    return q_hat


@_nvtx
def score_select(q_hat: torch.Tensor, k_cache: torch.Tensor, seq_lens: torch.Tensor, top_k: int,
                 *, sel_idx: torch.Tensor | None = None, scores: torch.Tensor | None = None,
                 workspace: torch.Tensor | None = None, aggregation: int = AGG_MAX,
                 dev_flags: torch.Tensor | None = None, stream=None,
                 params: SelectParams | None = None) -> torch.Tensor:
    """a2+a3 -> asyncspade_score_select.  q_hat fp32 [B, Hq, D]; k_cache bf16
    [B, Hkv, L, D] (strided, unit d-stride); seq_lens int32 [B].  Returns
    sel_idx int32 [B, Hkv, top_k] (ascending, -1 padded)."""
    p = params or select_params(q_hat, k_cache, top_k, aggregation)
    if sel_idx is None:
        sel_idx = torch.empty(p.batch, p.n_kv_heads, top_k, dtype=torch.int32,
                              device=q_hat.device)
    ws_bytes = 0
    if scores is None:
        ws_bytes = score_select_workspace(p)
        if workspace is None:
            workspace = _workspace(ws_bytes, q_hat.device)
        ws_bytes = workspace.numel() * workspace.element_size()
    _check(lib().asyncspade_score_select(ctypes.byref(p), _ptr(q_hat), _ptr(_u16(k_cache)),
                                         _ptr(seq_lens), _ptr(sel_idx), _ptr(scores),
                                         _ptr(workspace), ws_bytes, _ptr(dev_flags),
                                         _stream(stream)),
           "asyncspade_score_select")
    return sel_idx


@_nvtx
def sparse_decode(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                  seq_lens: torch.Tensor, sel_idx: torch.Tensor, *, n_fresh: int = 0,
                  sm_scale: float | None = None, out: torch.Tensor | None = None,
                  workspace: torch.Tensor | None = None, stream=None,
                  params: DecodeParams | None = None) -> torch.Tensor:
    """a4 -> asyncspade_sparse_decode.  q bf16 [B, Hq, D]; caches bf16
    [B, Hkv, L, D]; sel_idx int32 [B, Hkv, k].  Returns out fp32 [B, Hq, D]
    (or [Hq, B, D] when params.out_stride_b is set: head-major)."""
    p = params or decode_params(q, k_cache, v_cache, sel_idx.shape[-1], n_fresh, sm_scale)
    if out is None:
        B, Hq, D = q.shape
        dv = p.v_head_dim or D
        shape = (Hq, B, dv) if p.out_stride_b else (B, Hq, dv)
        out = torch.empty(shape, dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = _workspace(sparse_decode_workspace(p), q.device)
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(lib().asyncspade_sparse_decode(ctypes.byref(p), _ptr(_u16(q)), _ptr(_u16(k_cache)),
                                          _ptr(_u16(v_cache)), _ptr(seq_lens), _ptr(sel_idx),
                                          _ptr(out), _ptr(workspace), ws_bytes, _stream(stream)),
           "asyncspade_sparse_decode")
    return out


@_nvtx
def gather_filtered(k_cache: torch.Tensor, v_cache: torch.Tensor, seq_lens: torch.Tensor,
                    sel_idx: torch.Tensor, *, n_fresh: int = 0, k_out: torch.Tensor | None = None,
                    v_out: torch.Tensor | None = None, idx_out: torch.Tensor | None = None,
                    stream=None, params: DecodeParams | None = None):
    """The Cache Rank's payload -> asyncspade_gather_filtered: the selected
    K / V rows packed contiguously [B, Hkv, k, D] (bit-equal) and, if idx_out
    is given, the selection over the packed rows (j or -1)."""
    B, Hkv, L, D = k_cache.shape
    k = sel_idx.shape[-1]
    if k_out is None:
        k_out = torch.empty(B, Hkv, k, D, dtype=k_cache.dtype, device=k_cache.device)
    if v_out is None:
        v_out = torch.empty(B, Hkv, k, D, dtype=v_cache.dtype, device=v_cache.device)
    if k_out.shape != v_out.shape or k_out.stride() != v_out.stride() or k_out.stride(3) != 1 \
            or k_out.stride(2) != D or k_out.shape[2] != k:
        raise AsyncSpadeError("k_out / v_out: [B, Hkv, k, D] views with rows of D elements")
    # (b, h) blocks at k_out's strides: a [B, Hkv, k + 1, D] compact cache's first
    # k rows are a valid target
    osb, osh = ((0, 0) if k_out.is_contiguous() else (k_out.stride(0), k_out.stride(1)))
    p = params or DecodeParams(B, Hkv, Hkv, D, k, n_fresh, L, D ** -0.5, *k_cache.stride()[:3],
                               *v_cache.stride()[:3], osb, osh)
    _check(lib().asyncspade_gather_filtered(ctypes.byref(p), _ptr(_u16(k_cache)), _ptr(_u16(v_cache)),
                                            _ptr(seq_lens), _ptr(sel_idx), _ptr(_u16(k_out)),
                                            _ptr(_u16(v_out)), _ptr(idx_out), _stream(stream)),
           "asyncspade_gather_filtered")
    return k_out, v_out


# --------------------------------------------------------------------------- paged pools
def paged_kv(k_pages: torch.Tensor, block_table: torch.Tensor) -> PagedKV:
    """Geometry of a paged pool k_pages bf16 [num_pages, Hkv, page_size, D]
    (contiguous, HND) with block_table int32 [batch, max_pages_per_seq]."""
    n_pages, _, P, _ = k_pages.shape
    if not k_pages.is_contiguous() or not block_table.is_contiguous():
        raise AsyncSpadeError("the page pool and block table must be contiguous")
    return PagedKV(P, block_table.shape[1], n_pages)


@_nvtx
def score_select_paged(q_hat: torch.Tensor, k_pages: torch.Tensor, block_table: torch.Tensor,
                       seq_lens: torch.Tensor, top_k: int, max_seq_len: int, *,
                       sel_idx: torch.Tensor | None = None, scores: torch.Tensor | None = None,
                       workspace: torch.Tensor | None = None, aggregation: int = AGG_MAX,
                       dev_flags: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """a2+a3 over a paged K pool -> asyncspade_score_select_paged.  Returns
    sel_idx int32 [B, Hkv, top_k] of LOGICAL token positions."""
    B, Hq, D = q_hat.shape
    Hkv = k_pages.shape[1]
    p = SelectParams(B, Hq, Hkv, D, top_k, max_seq_len, aggregation, 0, 0, D)
    pk = paged_kv(k_pages, block_table)
    if sel_idx is None:
        sel_idx = torch.empty(B, Hkv, top_k, dtype=torch.int32, device=q_hat.device)
    ws_bytes = 0
    if scores is None:
        ws_bytes = score_select_workspace(p)
        if workspace is None:
            workspace = _workspace(ws_bytes, q_hat.device)
        ws_bytes = workspace.numel() * workspace.element_size()
    _check(lib().asyncspade_score_select_paged(ctypes.byref(p), ctypes.byref(pk), _ptr(q_hat),
                                               _ptr(_u16(k_pages)), _ptr(block_table),
                                               _ptr(seq_lens), _ptr(sel_idx), _ptr(scores),
                                               _ptr(workspace), ws_bytes, _ptr(dev_flags),
                                               _stream(stream)),
           "asyncspade_score_select_paged")
    return sel_idx


@_nvtx
def sparse_decode_paged(q: torch.Tensor, k_pages: torch.Tensor, v_pages: torch.Tensor,
                        block_table: torch.Tensor, seq_lens: torch.Tensor, sel_idx: torch.Tensor,
                        max_seq_len: int, *, n_fresh: int = 0, sm_scale: float | None = None,
                        out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                        stream=None) -> torch.Tensor:
    """a4 over paged K / V pools -> asyncspade_sparse_decode_paged."""
    B, Hq, D = q.shape
    Hkv = k_pages.shape[1]
    if sm_scale is None:
        sm_scale = D ** -0.5
    p = DecodeParams(B, Hq, Hkv, D, sel_idx.shape[-1], n_fresh, max_seq_len, sm_scale,
                     0, 0, D, 0, 0, D)
    pk = paged_kv(k_pages, block_table)
    if out is None:
        out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = _workspace(sparse_decode_workspace(p), q.device)
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(lib().asyncspade_sparse_decode_paged(ctypes.byref(p), ctypes.byref(pk), _ptr(_u16(q)),
                                                _ptr(_u16(k_pages)), _ptr(_u16(v_pages)),
                                                _ptr(block_table), _ptr(seq_lens), _ptr(sel_idx),
                                                _ptr(out), _ptr(workspace), ws_bytes,
                                                _stream(stream)),
           "asyncspade_sparse_decode_paged")
    return out


def page_pool(cache: torch.Tensor, page_size: int, generator: torch.Generator | None = None,
              spare_pages: int = 0):
    """Scatter a dense cache [B, Hkv, L, D] into a paged pool with a random
    page placement: returns (pool [B*L/P + spare, Hkv, P, D], block_table
    int32 [B, L/P]).  Data movement only (torch ops); used to build paged
    inputs for tests and the bench, not on the path."""
    B, Hkv, L, D = cache.shape
    if L % page_size:
        raise AsyncSpadeError("L must be a multiple of page_size")
    npp = L // page_size
    n_pages = B * npp + spare_pages
    perm = torch.randperm(n_pages, generator=generator)[:B * npp].to(torch.int32)
    block_table = perm.view(B, npp).to(cache.device)
    pool = torch.zeros(n_pages, Hkv, page_size, D, dtype=cache.dtype, device=cache.device)
    src = cache.view(B, Hkv, npp, page_size, D).permute(0, 2, 1, 3, 4).reshape(B * npp, Hkv,
                                                                                 page_size, D)
    pool[block_table.view(-1).long()] = src
    return pool, block_table


# --------------------------------------------------------------------------- Quest comparator
@_nvtx
def quest_summarize(k_cache: torch.Tensor, seq_lens: torch.Tensor, page_size: int, top_k: int,
                    n_q_heads: int, *, meta: torch.Tensor | None = None,
                    stream=None) -> torch.Tensor:
    """Page extremes of a dense K cache -> asyncspade_quest_summarize."""
    B, Hkv, L, D = k_cache.shape
    p = SelectParams(B, n_q_heads, Hkv, D, top_k, L, AGG_MAX, *k_cache.stride()[:3])
    if meta is None:
        meta = torch.empty(max(int(lib().asyncspade_quest_meta_bytes(ctypes.byref(p), page_size)),
                               256), dtype=torch.uint8, device=k_cache.device)
    _check(lib().asyncspade_quest_summarize(ctypes.byref(p), page_size, _ptr(_u16(k_cache)),
                                            _ptr(seq_lens), _ptr(meta), _stream(stream)),
           "asyncspade_quest_summarize")
    return meta


@_nvtx
def quest_select(q: torch.Tensor, meta: torch.Tensor, k_cache: torch.Tensor,
                 seq_lens: torch.Tensor, top_k: int, page_size: int, *,
                 sel_idx: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                 aggregation: int = AGG_MAX, dev_flags: torch.Tensor | None = None,
                 stream=None) -> torch.Tensor:
    """Quest page-bound selection -> asyncspade_quest_select.  q fp32
    [B, Hq, D]; returns token indices int32 [B, Hkv, top_k] (whole pages)."""
    B, Hq, D = q.shape
    _, Hkv, L, _ = k_cache.shape
    p = SelectParams(B, Hq, Hkv, D, top_k, L, aggregation, *k_cache.stride()[:3])
    if sel_idx is None:
        sel_idx = torch.empty(B, Hkv, top_k, dtype=torch.int32, device=q.device)
    if workspace is None:
        workspace = _workspace(int(lib().asyncspade_quest_select_workspace(ctypes.byref(p),
                                                                          page_size)), q.device)
    ws_bytes = workspace.numel() * workspace.element_size()
    _check(lib().asyncspade_quest_select(ctypes.byref(p), page_size, _ptr(q), _ptr(meta),
                                         _ptr(seq_lens), _ptr(sel_idx), _ptr(workspace), ws_bytes,
                                         _ptr(dev_flags), _stream(stream)),
           "asyncspade_quest_select")
    return sel_idx

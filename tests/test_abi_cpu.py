"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/asyncspade.h declares, and rejects invalid arguments
synchronously -- before anything could be enqueued."""
import ctypes
import os
import re

import pytest

import paper_2510_07486_b200 as asp
from paper_2510_07486_b200 import build as asp_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "asyncspade.h")


@pytest.fixture(scope="module")
def L():
    asp_build.build()
    return asp.lib()


def _declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(asyncspade_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = _declared_symbols()
    assert set(names) == set(asp.EXPORTED_SYMBOLS)
    for n in names:
        assert hasattr(L, n), n
    # and nothing else leaks out of the library
    out = os.popen(f"nm -D --defined-only {asp.LIB_PATH}").read()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert exported == set(names)


def test_version_and_status_strings(L):
    assert L.asyncspade_abi_version() == asp.ABI_VERSION
    for code, name in enumerate(["ASP_OK", "ASP_ERR_INVALID_ARGUMENT", "ASP_ERR_SHAPE",
                                 "ASP_ERR_UNSUPPORTED", "ASP_ERR_WORKSPACE", "ASP_ERR_CUDA"]):
        assert asp.status_string(code) == name
    assert asp.status_string(99) == "ASP_ERR_UNKNOWN"


FAKE = 0x10000  # 16-B aligned non-null "device" pointer: never dereferenced on error paths


def test_predict_validation(L):
    good = asp.PredictParams(2, 4, 16, 128, 0, 1e-2, 0)

    def call(p, win=FAKE, out=FAKE):
        return L.asyncspade_predict_query(ctypes.byref(p), win, out, None, None)

    assert call(good, win=None) == 1
    assert call(good, out=FAKE + 4) == 1                       # misaligned
    for bad in [asp.PredictParams(0, 4, 16, 128, 0, 1e-2, 0),
                asp.PredictParams(2, 4, 0, 128, 0, 1e-2, 0),
                asp.PredictParams(2, 4, 16, 128, 16, 1e-2, 0)]:  # ring_start out of range
        assert call(bad) == 2
    assert call(asp.PredictParams(2, 4, 16, 96, 0, 1e-2, 0)) == 3   # head_dim
    assert call(asp.PredictParams(2, 4, 33, 128, 0, 1e-2, 0)) == 3  # window
    assert call(asp.PredictParams(2, 4, 16, 128, 0, 1e-2, 3)) == 1  # unknown assembly
    assert call(asp.PredictParams(2, 4, 16, 128, 0, 1e-2, 1 << 9)) == 1
    assert call(asp.PredictParams(2, 4, 16, 128, 0, 1e-2, asp.NORM_NONE)) == 1  # needs SINGLE
    assert call(asp.PredictParams(2, 4, 16, 128, 0, float("nan"), 0)) == 1


def _sel(**kw):
    d = dict(batch=2, n_q_heads=32, n_kv_heads=8, head_dim=128, top_k=64, max_seq_len=1024,
             aggregation=0, k_stride_b=8 * 1024 * 128, k_stride_h=1024 * 128, k_stride_t=128)
    d.update(kw)
    return asp.SelectParams(*[d[f] for f, _ in asp.SelectParams._fields_])


def test_score_select_validation_and_workspace(L):
    def call(p, ws=FAKE, nbytes=1 << 40, q=FAKE, k=FAKE, sl=FAKE, idx=FAKE, scores=None):
        return L.asyncspade_score_select(ctypes.byref(p), q, k, sl, idx, scores, ws, nbytes,
                                         None, None)

    p = _sel()
    need = L.asyncspade_score_select_workspace(ctypes.byref(p))
    assert need >= 2 * 8 * 1024 * 4 and need % 256 == 0
    assert call(p, q=None) == 1
    assert call(p, k=FAKE + 2) == 1
    assert call(p, nbytes=need - 1) == 4
    assert call(p, ws=None) == 4
    assert call(p, ws=FAKE + 16) == 4                          # workspace must be 256-B aligned
    assert call(_sel(n_q_heads=30)) == 2
    assert call(_sel(top_k=0)) == 2
    assert call(_sel(n_q_heads=2048)) == 3                     # G = 256 (not built)
    assert call(_sel(head_dim=96, k_stride_t=96)) == 3          # head_dim 96 (not built)
    assert call(_sel(aggregation=2)) == 1
    assert call(_sel(k_stride_t=100)) == 2                     # shorter than a row
    assert call(_sel(k_stride_t=132)) == 1                     # not a multiple of 8 elements
    assert call(_sel(k_stride_h=1024 * 128 + 8)) == 3          # not a multiple of k_stride_t
    assert L.asyncspade_score_select_workspace(ctypes.byref(_sel(batch=0))) == 0


def _dec(**kw):
    d = dict(batch=2, n_q_heads=32, n_kv_heads=8, head_dim=128, top_k=64, n_fresh=1,
             max_seq_len=1024, sm_scale=128 ** -0.5, k_stride_b=8 * 1024 * 128, k_stride_h=1024 * 128,
             k_stride_t=128, v_stride_b=8 * 1024 * 128, v_stride_h=1024 * 128, v_stride_t=128,
             out_stride_b=0, out_stride_h=0, v_head_dim=0)
    d.update(kw)
    return asp.DecodeParams(*[d[f] for f, _ in asp.DecodeParams._fields_])


def test_sparse_decode_validation_and_workspace(L):
    def call(p, ws=FAKE, nbytes=1 << 40, out=FAKE, idx=FAKE):
        return L.asyncspade_sparse_decode(ctypes.byref(p), FAKE, FAKE, FAKE, FAKE, idx, out, ws,
                                          nbytes, None)

    p = _dec()
    need = L.asyncspade_sparse_decode_workspace(ctypes.byref(p))
    # one 256-entry chunk: [B][Hq][1][D + 2] fp32 partials
    assert need >= 2 * 32 * 1 * 130 * 4 and need % 256 == 0
    # 601 entries: three 256-entry chunks (rows of <= 384 entries are one item)
    need3 = L.asyncspade_sparse_decode_workspace(ctypes.byref(_dec(top_k=600)))
    assert need3 >= 2 * 32 * 3 * 130 * 4 and need3 % 256 == 0
    assert call(p, out=None) == 1
    assert call(p, idx=None) == 1
    assert call(p, nbytes=need - 1) == 4
    assert call(_dec(n_fresh=-1)) == 2
    assert call(_dec(n_q_heads=12)) == 2
    assert call(_dec(head_dim=80, k_stride_t=80, v_stride_t=80)) == 3
    # v_head_dim (ABI 2): > head_dim is a shape error; MLA 576 / 512 at G = 4 is built
    assert call(_dec(v_head_dim=256)) == 2
    mla = _dec(n_q_heads=32, n_kv_heads=8, head_dim=576, v_head_dim=512, k_stride_t=576,
               v_stride_t=576, k_stride_b=8 * 1024 * 576, k_stride_h=1024 * 576,
               v_stride_b=8 * 1024 * 576, v_stride_h=1024 * 576)
    # split-K partials of Dv = 512 values: [B][Hq][1][512 + 2] fp32
    assert L.asyncspade_sparse_decode_workspace(ctypes.byref(mla)) >= 2 * 32 * 514 * 4
    assert L.asyncspade_sparse_decode_workspace(ctypes.byref(_dec(head_dim=576, v_head_dim=448,
                                                                  k_stride_t=576, v_stride_t=576))) == 0
    assert call(_dec(v_stride_h=1004)) == 1
    assert call(_dec(sm_scale=float("nan"))) == 1
    assert call(_dec(max_seq_len=0)) == 2
    assert call(_dec(k_stride_h=1024 * 128 + 8)) == 3           # not a multiple of stride_t
    # output strides (ABI 2): both 0 (dense) or both set, >= 0, multiples of 4
    assert call(_dec(out_stride_b=128, out_stride_h=0)) == 2
    assert call(_dec(out_stride_b=-128, out_stride_h=256)) == 2
    assert call(_dec(out_stride_b=130, out_stride_h=256)) == 1


def test_synth_library_exports():
    """The bench/test input generator library loads and exports its two calls."""
    from paper_2510_07486_b200 import synth
    L = synth._dev_lib()
    assert hasattr(L, "asp_synth_kv") and hasattr(L, "asp_synth_query")


def test_paged_validation(L):
    """Paged entry points: page sizes 16..128 only, the block table must cover
    max_seq_len, the pool must stay below 2^31 rows, null pointers rejected."""
    sp = asp.SelectParams(2, 16, 8, 128, 64, 1024, 0, 0, 0, 128)
    dp = asp.DecodeParams(2, 16, 8, 128, 64, 0, 1024, 0.088, 0, 0, 128, 0, 0, 128)

    def sel(pk, bt=FAKE):
        return L.asyncspade_score_select_paged(ctypes.byref(sp), ctypes.byref(pk), FAKE, FAKE, bt,
                                               FAKE, FAKE, FAKE, None, 0, None, None)

    def dec(pk, bt=FAKE):
        return L.asyncspade_sparse_decode_paged(ctypes.byref(dp), ctypes.byref(pk), FAKE, FAKE,
                                                FAKE, bt, FAKE, FAKE, FAKE, None, 0, None)

    for fn in (sel, dec):
        assert fn(asp.PagedKV(8, 128, 256)) == 3                 # page size not built
        assert fn(asp.PagedKV(24, 64, 256)) == 3
        assert fn(asp.PagedKV(16, 32, 256)) == 2                 # 32 * 16 < max_seq_len
        assert fn(asp.PagedKV(16, 64, 0)) == 2
        assert fn(asp.PagedKV(128, 8, 1 << 22)) == 2             # pool rows >= 2^31
        assert fn(asp.PagedKV(16, 64, 256), bt=None) == 1
    assert L.asyncspade_score_select_paged(ctypes.byref(sp), None, FAKE, FAKE, FAKE, FAKE, FAKE,
                                           FAKE, None, 0, None, None) == 1
    # decode needs its workspace: a valid call shape without one is rejected as such
    assert dec(asp.PagedKV(16, 64, 256)) == 4


def test_predict_bf16_window_validation(L):
    """ASP_WINDOW_BF16 is built for the fast path only (2 <= W <= 16,
    masked-shared or single assembly)."""
    def call(W, flags):
        p = asp.PredictParams(2, 4, W, 128, 0, 1e-2, flags)
        return L.asyncspade_predict_query(ctypes.byref(p), FAKE, FAKE, None, None)

    assert call(32, asp.WINDOW_BF16) == 3
    assert call(1, asp.WINDOW_BF16) == 3
    assert call(8, asp.WINDOW_BF16 | asp.ASSEMBLY_PER_WINDOW) == 3
    assert call(8, asp.WINDOW_BF16 | (1 << 12)) == 1                 # unknown bit


def test_quest_group_validation(L):
    """The Quest comparator is built for G in {1, 2, 4, 8}: larger groups are
    refused on the host (ASP_ERR_UNSUPPORTED, zero workspace) -- the validation
    happens before anything could be enqueued."""
    ok = _sel(n_q_heads=64, top_k=64)                         # G = 8
    assert L.asyncspade_quest_select_workspace(ctypes.byref(ok), 16) > 0
    for G in (16, 32):
        p = _sel(n_q_heads=8 * G, top_k=64)
        assert L.asyncspade_quest_select_workspace(ctypes.byref(p), 16) == 0
        assert L.asyncspade_quest_select(ctypes.byref(p), 16, FAKE, FAKE, FAKE, FAKE, FAKE,
                                         1 << 40, None, None) == 3

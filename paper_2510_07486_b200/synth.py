"""Seeded synthetic inputs for the decode hot path (host / numpy side).

This module holds NO arithmetic of the method: it only draws the inputs the
paper's workload has:

* K, V ~ N(0, 1) rounded to bf16 (SPEC S:375 key/value generator);
* query windows follow SPEC's AR(1) trace q_t = 0.95 q_{t-1} + 0.05 xi_t
   for W steps; the current query q is step W, rounded to bf16.

Every value is a pure function of (seed, stream, global index), computed with
integer arithmetic plus IEEE round-to-nearest fp32 multiply/add only, so the
device generator in ``csrc/synth.cu`` reproduces it bit for bit (checked by
tests/test_gpu_parity.py::test_device_generator_matches_host).  Both the
oracle side (tests) and the CUDA side (tests, bench) draw from this one
definition; nothing here depends on either.

Normal deviates: Irwin-Hall(4) of four 16-bit lanes of a splitmix64 hash,
centred and scaled to unit variance (support +-3.46 sigma) -- an exactly
reproducible stand-in for Box-Muller, whose transcendental functions differ
between libm and CUDA.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
STREAM_K, STREAM_V, STREAM_Q = 1, 2, 3
NORM_SCALE = np.float32(1.0 / 37837.22668)   # 1 / std of a sum of four U{0..65535}
NORM_MEAN = 131070                            # 4 * 65535 / 2
AR_ALPHA = np.float32(0.95)
AR_SIGMA = np.float32(0.05)


# layer l of a layer-packed step uses seed + LAYER_SEED_STRIDE * l
LAYER_SEED_STRIDE = 7919

def base_seed(config_index: int, repetition: int = 0) -> int:
    """seed = 20251008 + 1000 * config_index + repetition."""
    return 20251008 + 1000 * config_index + repetition


def _splitmix64_scalar(x: int) -> int:
    z = (x + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int) -> int:
    return _splitmix64_scalar((seed ^ (stream << 48)) & M64)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def normal_from_index(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """fp32 N(0,1)-like deviate for each uint64 global index."""
    with np.errstate(over="ignore"):
        z = _splitmix64(np.uint64(stream_key(seed, stream)) + idx.astype(np.uint64))
    m = np.uint64(0xFFFF)
    s = ((z & m) + ((z >> np.uint64(16)) & m) + ((z >> np.uint64(32)) & m)
         + (z >> np.uint64(48))).astype(np.int64) - NORM_MEAN
    return s.astype(np.float32) * NORM_SCALE          # exact int->fp32, one RN multiply


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (finite inputs)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.asarray(h, np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def kv_rows(seed: int, stream: int, b: int, h: int, t0: int, t1: int, n_kv_heads: int,
            max_len: int, head_dim: int) -> np.ndarray:
    """bf16 bits [t1-t0, D] of K (stream 1) or V (stream 2) for GLOBAL batch b,
    GLOBAL kv head h, tokens [t0, t1)."""
    t = np.arange(t0, t1, dtype=np.uint64)[:, None]
    d = np.arange(head_dim, dtype=np.uint64)[None, :]
    idx = ((np.uint64(b) * np.uint64(n_kv_heads) + np.uint64(h)) * np.uint64(max_len) + t) \
        * np.uint64(head_dim) + d
    return f32_to_bf16_bits(normal_from_index(seed, stream, idx))


def kv_cache(seed: int, stream: int, batch: int, n_kv_heads: int, max_len: int, head_dim: int,
             b0: int = 0, h0: int = 0, n_kv_heads_global: int | None = None,
             batch_slice: int | None = None, head_slice: int | None = None) -> np.ndarray:
    """bf16 bits [B_s, H_s, L, D]; a shard (b0.., h0..) of the global tensor."""
    hg = n_kv_heads if n_kv_heads_global is None else n_kv_heads_global
    bs = batch if batch_slice is None else batch_slice
    hs = n_kv_heads if head_slice is None else head_slice
    out = np.empty((bs, hs, max_len, head_dim), np.uint16)
    for i in range(bs):
        for j in range(hs):
            out[i, j] = kv_rows(seed, stream, b0 + i, h0 + j, 0, max_len, hg, max_len, head_dim)
    return out


def query_trace(seed: int, batch: int, n_q_heads: int, window: int, head_dim: int,
                b0: int = 0, h0: int = 0, n_q_heads_global: int | None = None,
                batch_slice: int | None = None, head_slice: int | None = None):
    """AR(1) query trace: returns (window fp32 [B_s, H_s, W, D] in
    logical order oldest..newest, q bf16 bits [B_s, H_s, D] = step W)."""
    hg = n_q_heads if n_q_heads_global is None else n_q_heads_global
    bs = batch if batch_slice is None else batch_slice
    hs = n_q_heads if head_slice is None else head_slice
    T = window + 1
    b = np.arange(b0, b0 + bs, dtype=np.uint64)[:, None, None, None]
    h = np.arange(h0, h0 + hs, dtype=np.uint64)[None, :, None, None]
    t = np.arange(T, dtype=np.uint64)[None, None, :, None]
    d = np.arange(head_dim, dtype=np.uint64)[None, None, None, :]
    idx = ((b * np.uint64(hg) + h) * np.uint64(T) + t) * np.uint64(head_dim) + d
    xi = normal_from_index(seed, STREAM_Q, idx)
    qs = np.empty_like(xi)
    qs[:, :, 0] = xi[:, :, 0]
    for s in range(1, T):
        a = (AR_ALPHA * qs[:, :, s - 1]).astype(np.float32)
        e = (AR_SIGMA * xi[:, :, s]).astype(np.float32)
        qs[:, :, s] = (a + e).astype(np.float32)
    return np.ascontiguousarray(qs[:, :, :window]), f32_to_bf16_bits(qs[:, :, window])


# --------------------------------------------------------------------------- structured keys
# SURVEY §8(d) structured variants (test inputs only): heavy-hitter "needles"
# and an attention "sink", planted along the newest window query of
# the KV head's first q head, so they are known at generation time.
STREAM_NEEDLE = 4
N_NEEDLES = 32
NEEDLE_GAIN = 4.0        # needle rows: K += 4 sqrt(D) unit(Q_t)
SINK_GAIN = 8.0          # token 0:     K += 8 sqrt(D) unit(Q_t)


def needle_positions(seed: int, b: int, h: int, seq_len: int, n: int = N_NEEDLES) -> np.ndarray:
    """n distinct sorted positions in [1, seq_len) for GLOBAL (b, h): a
    counter-based draw (splitmix64 of (b, h, i)), duplicates skipped."""
    n = min(n, max(seq_len - 1, 0))
    key = stream_key(seed, STREAM_NEEDLE)
    out, seen, i = [], set(), 0
    while len(out) < n:
        z = _splitmix64_scalar((key + ((b * 65536 + h) << 20) + i) & M64)
        t = 1 + int(z % (seq_len - 1))
        if t not in seen:
            seen.add(t)
            out.append(t)
        i += 1
    return np.array(sorted(out), np.int64)


def structure_direction(seed: int, b: int, h: int, group: int, n_q_heads: int, window: int,
                        head_dim: int) -> np.ndarray:
    """fp32 [D]: sqrt(D) * unit(Q_t) for the newest window query of q head h*G
    (GLOBAL indices), the direction the needles and the sink are planted along."""
    win, _ = query_trace(seed, b + 1, n_q_heads, window, head_dim, b0=b, h0=h * group,
                         batch_slice=1, head_slice=1)
    qt = win[0, 0, window - 1].astype(np.float64)
    return (np.sqrt(head_dim) * qt / np.linalg.norm(qt)).astype(np.float32)


def structured_kv_rows(seed: int, b: int, h: int, seq_len: int, n_kv_heads: int, max_len: int,
                       head_dim: int, group: int, n_q_heads: int, window: int) -> np.ndarray:
    """K bf16 bits [seq_len, D] of GLOBAL (b, h) with the needles and the sink
    planted: row = bf16(float(row) + gain * direction) in fp32 (one RN add,
    then RNE -- what apply_structure_device does on the GPU)."""
    K = kv_rows(seed, STREAM_K, b, h, 0, max_len, n_kv_heads, max_len, head_dim)
    u = structure_direction(seed, b, h, group, n_q_heads, window, head_dim)
    rows = [(t, np.float32(NEEDLE_GAIN)) for t in needle_positions(seed, b, h, seq_len)]
    rows.append((0, np.float32(SINK_GAIN)))
    for t, gain in rows:
        d = (gain * u).astype(np.float32)
        K[t] = f32_to_bf16_bits((bf16_bits_to_f32(K[t]) + d).astype(np.float32))
    return K


def apply_structure_device(k_cache, seed: int, seq_len: int, n_kv_heads: int, group: int,
                           n_q_heads: int, window: int, b0: int = 0, h0: int = 0) -> None:
    """Plant the needles and the sink into a device K cache view [B_s, H_s, L, D]
    holding kv_cache(...) values of global (b0.., h0..), exactly as
    structured_kv_rows does on the host (directions computed on the host)."""
    import torch
    B, H, L, D = k_cache.shape
    for i in range(B):
        for j in range(H):
            b, h = b0 + i, h0 + j
            u = structure_direction(seed, b, h, group, n_q_heads, window, D)
            pos = needle_positions(seed, b, h, seq_len)
            d_needle = torch.from_numpy((np.float32(NEEDLE_GAIN) * u).astype(np.float32))
            d_sink = torch.from_numpy((np.float32(SINK_GAIN) * u).astype(np.float32))
            dev = k_cache.device
            p = torch.from_numpy(pos).to(dev)
            rows = k_cache[i, j].index_select(0, p).float() + d_needle.to(dev)
            k_cache[i, j].index_copy_(0, p, rows.to(torch.bfloat16))
            k_cache[i, j, 0] = (k_cache[i, j, 0].float() + d_sink.to(dev)).to(torch.bfloat16)


# --------------------------------------------------------------------------- device side
_synth_lib = None


def _dev_lib():
    """libasp_synth.so: the same generator as a CUDA kernel (bench/test support)."""
    global _synth_lib
    if _synth_lib is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libasp_synth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python -m paper_2510_07486_b200.build`")
        L = ctypes.CDLL(path)
        i, ll, u64, vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_uint64, ctypes.c_void_p
        L.asp_synth_kv.argtypes = [u64, vp, i, i, i, i, i, i, i, ll, ll, ll, vp]
        L.asp_synth_kv.restype = i
        L.asp_synth_query.argtypes = [u64, vp, vp, i, i, i, i, i, i, i, vp]
        L.asp_synth_query.restype = i
        L.asp_synth_forward.argtypes = [vp, ll, vp, i, vp]
        L.asp_synth_forward.restype = i
        _synth_lib = L
    return _synth_lib


def fill_kv_device(cache, seed: int, stream_id: int, b0: int = 0, h0: int = 0,
                   n_kv_heads_global: int | None = None, stream=None) -> None:
    """Fill a bf16 torch cache view [B_s, H_s, L, D] (unit d-stride) on the GPU
    with kv_cache(...) values; L is the view's token extent."""
    import torch
    bs, hs, L, D = cache.shape
    hg = hs if n_kv_heads_global is None else n_kv_heads_global
    st = stream if stream is not None else torch.cuda.current_stream()
    sb, sh, stt, sd = cache.stride()
    assert sd == 1
    rc = _dev_lib().asp_synth_kv(stream_key(seed, stream_id), cache.data_ptr(), bs, hs, L, D,
                                 b0, h0, hg, sb, sh, stt, st.cuda_stream)
    if rc != 0:
        raise RuntimeError(f"asp_synth_kv failed: cuda error {rc}")


def fill_query_device(window, q, seed: int, b0: int = 0, h0: int = 0,
                      n_q_heads_global: int | None = None, stream=None) -> None:
    """Fill window fp32 [B_s, H_s, W, D] and q bf16 [B_s, H_s, D] (contiguous)
    with query_trace(...) values on the GPU."""
    import torch
    bs, hs, W, D = window.shape
    assert window.is_contiguous() and q.is_contiguous()
    hg = hs if n_q_heads_global is None else n_q_heads_global
    st = stream if stream is not None else torch.cuda.current_stream()
    rc = _dev_lib().asp_synth_query(stream_key(seed, STREAM_Q), window.data_ptr(), q.data_ptr(),
                                    bs, hs, W, D, b0, h0, hg, st.cuda_stream)
    if rc != 0:
        raise RuntimeError(f"asp_synth_query failed: cuda error {rc}")


# Qwen3-8B per-layer parameters (Table 1, head_dim 128): q/o 4096x4096,
# k/v 4096x1024, MLP 3 x 4096x12288 -> 192.9 M params, 386 MB bf16.
QWEN3_8B_LAYER_PARAMS = 2 * 4096 * 4096 + 2 * 4096 * 1024 + 3 * 4096 * 12288
# Qwen3-32B (Table 1, head_dim 128): q/o 5120x8192, k/v 5120x1024, MLP
# 3 x 5120x25600 -> 487.6 M params, 975 MB bf16 per layer (1/P of it per GPU
# under P-way tensor parallelism)
QWEN3_32B_LAYER_PARAMS = 2 * 5120 * 8192 + 2 * 5120 * 1024 + 3 * 5120 * 25600


def synthetic_forward(weights, sink, stream=None) -> None:
    """The synthetic forward of config [4]: one streaming read of `weights`
    (a uint8/bf16 device tensor) on `stream`."""
    import torch
    st = stream if stream is not None else torch.cuda.current_stream()
    n_sm = torch.cuda.get_device_properties(weights.device).multi_processor_count
    nbytes = weights.numel() * weights.element_size()
    rc = _dev_lib().asp_synth_forward(weights.data_ptr(), nbytes - nbytes % 16, sink.data_ptr(),
                                      n_sm, st.cuda_stream)
    if rc != 0:
        raise RuntimeError(f"asp_synth_forward failed: cuda error {rc}")

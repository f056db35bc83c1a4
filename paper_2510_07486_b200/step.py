"""DecodeStep -- one attention layer's AsyncSpade decode step on one GPU.

The public "whole path" API: it owns the device buffers of one (possibly
KV-head-sharded) layer and runs a1 -> a2+a3 -> a4 through the C ABI
(predict_query, score_select, sparse_decode), optionally replayed as a CUDA
graph.  torch is used only to allocate memory and provide the stream.

Layer packing (the paper's depth-wise parallelism,
P:247-249): with `layers = P_l` the buffers of P_l consecutive layers are
stacked along the batch axis ([P_l * B, ...], layer-major), so ONE launch of
each kernel predicts, scores, selects and attends for all P_l layers -- the
predicted queries of every layer are available together, and every row is
independent, so a packed step reproduces the per-layer steps bit for bit.

Sharding (§8(e) of SURVEY.md): a shard owns KV heads
[h0, h0 + n_kv_heads) and the matching q heads for every batch row.  Every
kernel's per-row arithmetic depends only on the row, so a shard reproduces
the matching slice of the unsharded result bit for bit.
"""
from __future__ import annotations

import torch

from . import (append, decode_params, predict_params, predict_query, score_select, select_params,
               sparse_decode, score_select_workspace, sparse_decode_workspace)
from . import synth
from .configs import Config


class DecodeStep:
    def __init__(self, cfg: Config, device="cuda", *, kv_heads: tuple[int, int] | None = None,
                 n_fresh: int = 0, eps: float = 1e-2, flags: int = 0, keep_scores: bool = False,
                 layers: int = 1, window_dtype: torch.dtype = torch.float32,
                 batch_range: tuple[int, int] | None = None, out_head_major: bool = False):
        self.cfg = cfg
        self.layers = layers
        self.device = torch.device(device)
        h0, hn = kv_heads if kv_heads is not None else (0, cfg.n_kv_heads)
        self.h0, self.n_kv = h0, hn
        G = cfg.group
        self.q0, self.n_q = h0 * G, hn * G
        W, D, L = cfg.window, cfg.head_dim, cfg.seq_len
        # batch rows [b0, b0 + n_b) of the global batch (a batch-split shard, §8(e))
        self.b0, self.n_b = batch_range if batch_range is not None else (0, cfg.batch)
        B = self.n_b * layers                      # layer-major packing along the batch axis
        dev = self.device
        self.n_fresh, self.eps, self.flags = n_fresh, eps, flags
        self.ring_start = 0
        self.window = torch.empty(B, self.n_q, W, D, dtype=window_dtype, device=dev)
        self.q = torch.empty(B, self.n_q, D, dtype=torch.bfloat16, device=dev)
        self.k_cache = torch.empty(B, hn, L, D, dtype=torch.bfloat16, device=dev)
        # absorbed MLA (v_head_dim < head_dim): the values are the latent part of
        # the key rows -- one cache, read once
        self.mla = bool(cfg.v_head_dim) and cfg.v_head_dim != D
        self.dv = cfg.v_head_dim or D
        self.v_cache = (self.k_cache if self.mla else
                        torch.empty(B, hn, L, D, dtype=torch.bfloat16, device=dev))
        self.seq_lens = torch.full((B,), L, dtype=torch.int32, device=dev)
        self.q_hat = torch.empty(B, self.n_q, D, dtype=torch.float32, device=dev)
        self.sel_idx = torch.empty(B, hn, cfg.top_k, dtype=torch.int32, device=dev)
        # out [B, n_q, Dv], or head-major [n_q, B, Dv]: a KV-head shard's block of
        # the gathered [Hq, B, Dv] output (the gather is a concatenation)
        self.out_head_major = out_head_major
        self.out = (torch.empty(self.n_q, B, self.dv, dtype=torch.float32, device=dev)
                    if out_head_major else
                    torch.empty(B, self.n_q, self.dv, dtype=torch.float32, device=dev))
        self.dev_flags = torch.zeros(1, dtype=torch.int32, device=dev)
        self.scores = (torch.empty(B, hn, L, dtype=torch.float32, device=dev)
                       if keep_scores else None)
        self.p_pred = predict_params(self.window, eps, flags, 0)
        self.p_sel = select_params(self.q_hat, self.k_cache, cfg.top_k)
        self.p_dec = decode_params(self.q, self.k_cache, self.v_cache, cfg.top_k, n_fresh,
                                   v_head_dim=cfg.v_head_dim if self.mla else 0,
                                   out_head_major=out_head_major)
        self.ws_sel = torch.empty(max(score_select_workspace(self.p_sel), 256), dtype=torch.uint8,
                                  device=dev)
        self.ws_dec = torch.zeros(max(sparse_decode_workspace(self.p_dec), 256),
                                  dtype=torch.uint8, device=dev)
        # one CUDA graph per ring position: the predict launch bakes ring_start
        # into its parameters, so append() (which advances it) selects another
        # graph instead of replaying a stale one
        self.graphs: dict[int, torch.cuda.CUDAGraph] = {}

    @property
    def graph(self):
        return self.graphs.get(self.ring_start)

    # ------------------------------------------------------------------ inputs
    def fill_synthetic(self, seed: int | None = None) -> None:
        """Seeded synthetic inputs of the config's shape: the
        values of global heads [h0, h0+n) -- identical on any sharding."""
        cfg = self.cfg
        seed = synth.base_seed(cfg.index) if seed is None else seed
        B = self.n_b
        for layer in range(self.layers):
            sd = seed + synth.LAYER_SEED_STRIDE * layer
            rows = slice(layer * B, (layer + 1) * B)
            synth.fill_kv_device(self.k_cache[rows], sd, synth.STREAM_K, self.b0, self.h0,
                                 cfg.n_kv_heads)
            if not self.mla:
                synth.fill_kv_device(self.v_cache[rows], sd, synth.STREAM_V, self.b0, self.h0,
                                     cfg.n_kv_heads)
            if self.window.dtype == torch.float32:
                synth.fill_query_device(self.window[rows], self.q[rows].view(torch.int16), sd,
                                        self.b0, self.q0, cfg.n_q_heads)
            else:                                          # a bf16 ring: the rounded trace
                w32 = torch.empty(self.window[rows].shape, dtype=torch.float32, device=self.device)
                synth.fill_query_device(w32, self.q[rows].view(torch.int16), sd, self.b0,
                                        self.q0, cfg.n_q_heads)
                self.window[rows].copy_(w32)
        self.ring_start = 0
        self.p_pred.ring_start = 0

    # ------------------------------------------------------------------ the path
    def run(self, stream=None) -> None:
        """a1 -> a2+a3 -> a4 on `stream` (default: current)."""
        predict_query(self.window, self.q_hat, dev_flags=self.dev_flags.view(torch.int32),
                      stream=stream, params=self.p_pred)
        score_select(self.q_hat, self.k_cache, self.seq_lens, self.cfg.top_k,
                     sel_idx=self.sel_idx, scores=self.scores, workspace=self.ws_sel,
                     dev_flags=self.dev_flags, stream=stream, params=self.p_sel)
        sparse_decode(self.q, self.k_cache, self.v_cache, self.seq_lens, self.sel_idx,
                      out=self.out, workspace=self.ws_dec, stream=stream, params=self.p_dec)

    def capture(self) -> torch.cuda.CUDAGraph:
        """Record run() into a CUDA graph for the current ring position
        (warm-up launch first).  Buffers are fixed, so a graph stays valid
        across fill_synthetic() / append(); append() moves to the graph of
        the next ring position (captured on first use)."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.run()
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run()
        self.graphs[self.ring_start] = g
        return g

    def replay(self) -> None:
        g = self.graph
        if g is None:
            g = self.capture()
        g.replay()

    # ------------------------------------------------------------------ a0: window push
    def append(self, q_t: torch.Tensor, k_new: torch.Tensor | None = None,
               v_new: torch.Tensor | None = None, pos: torch.Tensor | None = None,
               stream=None) -> None:
        """a0 in one kernel (asyncspade_append): q_t fp32 [B, n_q, D] becomes the
        newest window entry and (rounded to bf16) the current query; the new
        K / V rows [B, n_kv, D] land at pos[b]."""
        slot = self.ring_start
        append(q_t, self.window, slot, q_cur=self.q, k_new=k_new, v_new=v_new,
               k_cache=self.k_cache if k_new is not None else None,
               v_cache=self.v_cache if v_new is not None else None, pos=pos, stream=stream)
        self.ring_start = (slot + 1) % self.cfg.window
        self.p_pred.ring_start = self.ring_start

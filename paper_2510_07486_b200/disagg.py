"""Dual-rank disaggregation: the paper's Inference Rank
and Cache Rank (Fig. 4; SPEC duo-rank-pipeline S:502-608).

    Inference Rank                          Cache Rank (full KV cache + query windows)
    step t: [recv sel(t)] attention over     recv pack(t) = (q_t, k_t, v_t)
            sel(t) U its fresh token(s)      a0 append -> a1 predict q_hat(t+1)
            ... rest of the layer ...        -> a2/a3 score + top-k -> gather_filtered
            send pack(t) --------------->    send sel(t+1) = selected K/V rows
            <------------------------------

The Cache Rank's selection for step t+1 runs while the Inference Rank
finishes step t and starts t+1, so selection leaves the inference critical
path; the Inference Rank only attends over the k selected rows it receives
plus the newest token (n_fresh = 1, reading R12), which the Cache Rank's
selection cannot contain yet.  Every compute step is a library kernel
(asyncspade_append, _predict_query, _score_select, _gather_filtered,
_sparse_decode); this module only moves tensors.  The transport is
torch.distributed point-to-point (NCCL over NVLink between two GPUs; the
tests run both ranks on one GPU over gloo with host staging).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import (DecodeParams, gather_filtered, predict_query, score_select, sparse_decode,
               sparse_decode_workspace)
from .configs import Config
from .step import DecodeStep


class Transport:
    """Point-to-point sends of device tensors.  NCCL moves them directly;
    other backends (gloo) stage through pinned host buffers."""

    def __init__(self, peer: int, group=None):
        self.peer, self.group = peer, group
        self.staged = dist.get_backend(group) != "nccl"

    def send(self, t: torch.Tensor) -> None:
        if self.staged:                           # raw bytes: bit-exact for every dtype
            if t.is_cuda:
                torch.cuda.current_stream(t.device).synchronize()
            dist.send(t.contiguous().view(torch.uint8).cpu(), self.peer, group=self.group)
        else:
            dist.send(t, self.peer, group=self.group)

    def recv(self, t: torch.Tensor) -> None:
        if self.staged:
            h = torch.empty(t.contiguous().view(torch.uint8).shape, dtype=torch.uint8)
            dist.recv(h, self.peer, group=self.group)
            t.copy_(h.to(t.device).view(t.dtype).view(t.shape))
        else:
            dist.recv(t, self.peer, group=self.group)


class CacheRank:
    """Holds the full caches and windows of one layer pack; per step: takes the
    Inference Rank's pack, appends it, selects for the NEXT step and returns
    the selected K/V rows (bit-equal to the cache rows)."""

    def __init__(self, cfg: Config, device, transport: Transport, layers: int = 1):
        self.cfg, self.io = cfg, transport
        self.step = DecodeStep(cfg, device, layers=layers)
        st = self.step
        B = st.q.shape[0]
        self.q_t = torch.empty(B, st.n_q, cfg.head_dim, dtype=torch.float32, device=st.device)
        self.kv_t = torch.empty(2, B, st.n_kv, cfg.head_dim, dtype=torch.bfloat16, device=st.device)
        self.pos = torch.sub(st.seq_lens, 1)       # the newest slot (lengths held fixed)
        self.k_sel = torch.empty(B, st.n_kv, cfg.top_k, cfg.head_dim, dtype=torch.bfloat16,
                                 device=st.device)
        self.v_sel = torch.empty_like(self.k_sel)
        self.i_sel = torch.empty(B, st.n_kv, cfg.top_k, dtype=torch.int32, device=st.device)

    def select_and_gather(self) -> None:
        st = self.step
        predict_query(st.window, st.q_hat, dev_flags=st.dev_flags, params=st.p_pred)
        score_select(st.q_hat, st.k_cache, st.seq_lens, self.cfg.top_k, sel_idx=st.sel_idx,
                     workspace=st.ws_sel, dev_flags=st.dev_flags, params=st.p_sel)
        # the newest token is the Inference Rank's own (n_fresh = 1): packed rows
        # at or past it are marked -1 in the packed selection
        gather_filtered(st.k_cache, st.v_cache, st.seq_lens, st.sel_idx, n_fresh=1,
                        k_out=self.k_sel, v_out=self.v_sel, idx_out=self.i_sel)

    def send_selection(self) -> None:
        self.io.send(self.k_sel)
        self.io.send(self.v_sel)
        self.io.send(self.i_sel)

    def prime(self) -> None:
        """Selection for the first step (from the windows as they stand)."""
        self.select_and_gather()
        self.send_selection()

    def serve(self, send: bool = True) -> None:
        """One step: receive pack(t), append it, select for t+1 and (unless it
        is the last step) send sel(t+1)."""
        self.io.recv(self.q_t)
        self.io.recv(self.kv_t)
        self.step.append(self.q_t, self.kv_t[0], self.kv_t[1], self.pos)
        self.select_and_gather()
        if send:
            self.send_selection()


class InferenceRank:
    """Attends over the received selection plus its own newest token; sends
    each step's (q_t, k_t, v_t) to the Cache Rank."""

    def __init__(self, cfg: Config, device, transport: Transport, n_q: int, n_kv: int,
                 batch: int):
        self.cfg, self.io = cfg, transport
        dev = torch.device(device)
        D, k = cfg.head_dim, cfg.top_k
        # the compact cache: k received rows + the fresh token at row k
        self.k_c = torch.zeros(batch, n_kv, k + 1, D, dtype=torch.bfloat16, device=dev)
        self.v_c = torch.zeros_like(self.k_c)
        # contiguous receive buffers (point-to-point needs dense tensors); the
        # rows are then placed ahead of the fresh token
        self.k_r = torch.empty(batch, n_kv, k, D, dtype=torch.bfloat16, device=dev)
        self.v_r = torch.empty_like(self.k_r)
        self.lens = torch.full((batch,), k + 1, dtype=torch.int32, device=dev)
        self.idx = torch.empty(batch, n_kv, k, dtype=torch.int32, device=dev)   # packed selection
        self.q = torch.empty(batch, n_q, D, dtype=torch.bfloat16, device=dev)
        self.out = torch.empty(batch, n_q, D, dtype=torch.float32, device=dev)
        self.p = DecodeParams(batch, n_q, n_kv, D, k, 1, k + 1, D ** -0.5,
                              *self.k_c.stride()[:3], *self.v_c.stride()[:3])
        self.ws = torch.empty(max(sparse_decode_workspace(self.p), 256), dtype=torch.uint8,
                              device=dev)

    def step(self, q_t: torch.Tensor, kv_t: torch.Tensor) -> torch.Tensor:
        """Decode step t: q_t fp32 [B, Hq, D] (the current query), kv_t bf16
        [2, B, Hkv, D] (the new token).  Returns the attention output."""
        k = self.cfg.top_k
        self.io.recv(self.k_r)                     # sel(t), computed from pack(t-1)
        self.io.recv(self.v_r)
        self.io.recv(self.idx)
        self.k_c[:, :, :k].copy_(self.k_r)
        self.v_c[:, :, :k].copy_(self.v_r)
        self.k_c[:, :, k].copy_(kv_t[0])
        self.v_c[:, :, k].copy_(kv_t[1])
        self.q.copy_(q_t)
        sparse_decode(self.q, self.k_c, self.v_c, self.lens, self.idx, out=self.out,
                      workspace=self.ws, params=self.p)
        self.io.send(q_t)                          # pack(t) -> the Cache Rank
        self.io.send(kv_t)
        return self.out

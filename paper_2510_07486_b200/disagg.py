"""Dual-rank disaggregation: the paper's Inference Rank
and Cache Rank (Fig. 4; SPEC duo-rank-pipeline S:502-608).

    Inference Rank                          Cache Rank (full KV cache + query windows)
    step t: [sel(t) in?] attention over      recv pack(t) = (q_t, k_t, v_t)
            sel(t) U its fresh token         a0 append -> a1 predict q_hat(t+1)
            ... rest of the layer ...        -> a2/a3 score + top-k -> gather_filtered
            send pack(t) --------------->    send sel(t+1) = selected K/V rows
            <------------------------------

The Cache Rank's selection for step t+1 runs while the Inference Rank
finishes step t and starts t+1, so selection leaves the inference critical
path; the Inference Rank only attends over the k selected rows it receives
plus the newest token (n_fresh = 1, reading R12), which the Cache Rank's
selection cannot contain yet.

Every compute step is a library kernel (asyncspade_append, _predict_query,
_score_select, _gather_filtered, _sparse_decode); this module only moves
tensors, and nothing is copied or cast by torch on the Inference Rank's path:
the Cache Rank gathers the selected rows straight into the Inference Rank's
compact-cache layout [B][Hkv][k + 1][D] (row k is the receiver's own fresh
token), the receive lands in that cache, and one asyncspade_append writes the
fresh K / V row and the bf16 current query.

Stall policy ("stall_policy default = wait ... reuse-previous
offered"): when the Cache Rank is late, the Inference Rank either waits for
sel(t) ("wait") or attends with the newest selection it already holds
("reuse"; the late one is taken at the next step -- the newest completed
selection always wins).  The transport is torch.distributed point-to-point:
NCCL over NVLink between two GPUs, or gloo with raw-byte host staging (tests:
both ranks on one GPU).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import (DecodeParams, append, gather_filtered, predict_query, score_select,
               sparse_decode, sparse_decode_workspace)
from .configs import Config
from .step import DecodeStep


class _Pending:
    """A posted receive (NCCL: in place; gloo: into a host staging buffer)."""

    def __init__(self, work, t: torch.Tensor, host: torch.Tensor | None):
        self.work, self.t, self.host = work, t, host

    def done(self) -> bool:
        return self.work.is_completed()

    def finish(self) -> None:
        self.work.wait()
        if self.host is not None:
            self.t.view(torch.uint8).view(-1).copy_(self.host.to(self.t.device))


class Transport:
    """Point-to-point moves of device tensors.  NCCL moves them directly;
    other backends (gloo) stage raw bytes through host buffers (bit-exact for
    every dtype).  Sends and receives may use separate process groups: NCCL
    serialises a communicator's point-to-point operations on one stream, so
    the Inference Rank's posted receive of sel(t+1) would otherwise block its
    own send of pack(t) -- which the Cache Rank needs before it can send
    sel(t+1).  One group per direction keeps the two streams independent."""

    def __init__(self, peer: int, group=None, recv_group=None):
        self.peer, self.group = peer, group
        self.recv_group = group if recv_group is None else recv_group
        self.staged = dist.get_backend(group) != "nccl"

    @staticmethod
    def _bytes(t: torch.Tensor) -> torch.Tensor:
        return t.view(torch.uint8).view(-1)

    def send(self, t: torch.Tensor) -> None:
        if not t.is_contiguous():
            raise ValueError("point-to-point sends need contiguous tensors")
        if self.staged:
            if t.is_cuda:
                torch.cuda.current_stream(t.device).synchronize()
            dist.send(self._bytes(t).cpu(), self.peer, group=self.group)
        else:
            dist.send(t, self.peer, group=self.group)

    def irecv(self, t: torch.Tensor) -> _Pending:
        if not t.is_contiguous():
            raise ValueError("point-to-point receives need contiguous tensors")
        if self.staged:
            h = torch.empty(t.numel() * t.element_size(), dtype=torch.uint8)
            return _Pending(dist.irecv(h, self.peer, group=self.recv_group), t, h)
        return _Pending(dist.irecv(t, self.peer, group=self.recv_group), t, None)

    def recv(self, t: torch.Tensor) -> None:
        self.irecv(t).finish()


class CacheRank:
    """Holds the full caches and windows of one layer pack; per step: takes the
    Inference Rank's pack, appends it, selects for the NEXT step and returns
    the selected K/V rows (bit-equal to the cache rows) in the receiver's
    compact-cache layout."""

    def __init__(self, cfg: Config, device, transport: Transport, layers: int = 1):
        self.cfg, self.io = cfg, transport
        self.step = DecodeStep(cfg, device, layers=layers)
        st = self.step
        B, k, D = st.q.shape[0], cfg.top_k, cfg.head_dim
        self.q_t = torch.empty(B, st.n_q, D, dtype=torch.float32, device=st.device)
        self.kv_t = torch.empty(2, B, st.n_kv, D, dtype=torch.bfloat16, device=st.device)
        self.pos = torch.sub(st.seq_lens, 1)       # the newest slot (lengths held fixed)
        # [B][Hkv][k + 1][D]: the receiver's compact caches (row k: its fresh token)
        self.k_sel = torch.zeros(B, st.n_kv, k + 1, D, dtype=torch.bfloat16, device=st.device)
        self.v_sel = torch.zeros_like(self.k_sel)
        self.i_sel = torch.empty(B, st.n_kv, k, dtype=torch.int32, device=st.device)
        self.sent = []                             # global selections sent (tests / audit)

    def select_and_gather(self) -> None:
        st, k = self.step, self.cfg.top_k
        predict_query(st.window, st.q_hat, dev_flags=st.dev_flags, params=st.p_pred)
        score_select(st.q_hat, st.k_cache, st.seq_lens, k, sel_idx=st.sel_idx,
                     workspace=st.ws_sel, dev_flags=st.dev_flags, params=st.p_sel)
        # the newest token is the Inference Rank's own (n_fresh = 1): packed rows
        # at or past it are marked -1 in the packed selection
        gather_filtered(st.k_cache, st.v_cache, st.seq_lens, st.sel_idx, n_fresh=1,
                        k_out=self.k_sel[:, :, :k], v_out=self.v_sel[:, :, :k],
                        idx_out=self.i_sel)

    def send_selection(self, keep: bool = False) -> None:
        if keep:
            self.sent.append(self.step.sel_idx.cpu().clone())
        self.io.send(self.k_sel)
        self.io.send(self.v_sel)
        self.io.send(self.i_sel)

    def prime(self, keep: bool = False) -> None:
        """Selection for the first step (from the windows as they stand)."""
        self.select_and_gather()
        self.send_selection(keep)

    def serve(self, keep: bool = False, delay_s: float = 0.0) -> None:
        """One step: receive pack(t), append it, select for t+1, send sel(t+1)
        (after `delay_s`: tests of a late Cache Rank)."""
        self.io.recv(self.q_t)
        self.io.recv(self.kv_t)
        self.step.append(self.q_t, self.kv_t[0], self.kv_t[1], self.pos)
        self.select_and_gather()
        if delay_s:
            import time
            torch.cuda.current_stream(self.step.device).synchronize()
            time.sleep(delay_s)
        self.send_selection(keep)


class _StagedReceiver:
    """gloo: a background thread keeps a receive of the next selection posted
    (gloo completes a receive only inside wait(), so is_completed() cannot be
    polled) and queues the host copies; done() / finish() mirror _Pending."""

    def __init__(self, io: "Transport", shapes):
        import queue
        import threading
        self.io, self.q = io, queue.Queue()
        self.sizes = [int(torch.Size(sh).numel()) * es for sh, es in shapes]
        self.stop = False
        # one credit per selection the Cache Rank owes (the first, then one per
        # pack): the thread never posts a receive nobody will answer
        self.credits = threading.Semaphore(1)
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def expect_one(self) -> None:
        self.credits.release()

    def close(self) -> None:
        self.stop = True
        self.credits.release()
        self.th.join(timeout=30)

    def _run(self):
        while True:
            self.credits.acquire()
            if self.stop:
                return
            hs = []
            for n in self.sizes:
                h = torch.empty(n, dtype=torch.uint8)
                dist.recv(h, self.io.peer, group=self.io.recv_group)
                hs.append(h)
            self.q.put(hs)

    def done(self) -> bool:
        return not self.q.empty()

    def take(self, targets) -> None:
        hs = self.q.get()
        for t, h in zip(targets, hs):
            t.view(torch.uint8).view(-1).copy_(h.to(t.device))


class InferenceRank:
    """Attends over the received selection plus its own newest token; sends
    each step's (q_t, k_t, v_t) to the Cache Rank.  Two compact caches: the
    selection in use, and the one the next selection is received into."""

    def __init__(self, cfg: Config, device, transport: Transport, n_q: int, n_kv: int,
                 batch: int, stall_policy: str = "wait"):
        if stall_policy not in ("wait", "reuse"):
            raise ValueError("stall_policy: 'wait' or 'reuse'")
        self.cfg, self.io, self.policy = cfg, transport, stall_policy
        dev = torch.device(device)
        D, k = cfg.head_dim, cfg.top_k
        self.k_c = [torch.zeros(batch, n_kv, k + 1, D, dtype=torch.bfloat16, device=dev)
                    for _ in range(2)]
        self.v_c = [torch.zeros_like(self.k_c[0]) for _ in range(2)]
        self.idx = [torch.empty(batch, n_kv, k, dtype=torch.int32, device=dev) for _ in range(2)]
        self.lens = torch.full((batch,), k + 1, dtype=torch.int32, device=dev)
        self.pos = torch.full((batch,), k, dtype=torch.int32, device=dev)   # the fresh row
        self.q = torch.empty(batch, n_q, D, dtype=torch.bfloat16, device=dev)
        self.out = torch.empty(batch, n_q, D, dtype=torch.float32, device=dev)
        self.p = DecodeParams(batch, n_q, n_kv, D, k, 1, k + 1, D ** -0.5,
                              *self.k_c[0].stride()[:3], *self.v_c[0].stride()[:3], 0, 0)
        self.ws = torch.empty(max(sparse_decode_workspace(self.p), 256), dtype=torch.uint8,
                              device=dev)
        self.cur = -1                      # compact cache in use (-1: none yet)
        self.received = 0                  # selections installed so far
        self.used = []                     # per step: which selection (0-based) was used
        self.packs = 0                     # packs sent (the Cache Rank answers each)
        self.rx = None
        if self.io.staged:
            self.rx = _StagedReceiver(self.io, [(t.shape, t.element_size())
                                                for t in (self.k_c[0], self.v_c[0], self.idx[0])])
        self._post()

    def _post(self) -> None:
        nxt = 1 if self.cur == 0 else 0
        self.spare = nxt
        if self.rx is None:
            self.pending = [self.io.irecv(self.k_c[nxt]), self.io.irecv(self.v_c[nxt]),
                            self.io.irecv(self.idx[nxt])]

    def _arrived(self) -> bool:
        return self.rx.done() if self.rx is not None else all(pr.done() for pr in self.pending)

    def _install(self) -> None:
        if self.rx is not None:
            self.rx.take([self.k_c[self.spare], self.v_c[self.spare], self.idx[self.spare]])
        else:
            for pr in self.pending:
                pr.finish()
        self.cur = self.spare
        self.received += 1
        self._post()

    def step(self, q_t: torch.Tensor, kv_t: torch.Tensor) -> torch.Tensor:
        """Decode step t: q_t fp32 [B, Hq, D] (the current query), kv_t bf16
        [2, B, Hkv, D] (the new token).  Returns the attention output."""
        if self.cur < 0 or self.policy == "wait":
            self._install()                            # sel(t): wait for it
        while self._arrived():                         # reuse: take the newest arrived
            self._install()
        self.used.append(self.received - 1)
        c = self.cur
        # a0 on this rank: bf16(q_t) -> q, the fresh K / V row -> compact row k
        append(q_t, None, 0, q_cur=self.q, k_new=kv_t[0], v_new=kv_t[1], k_cache=self.k_c[c],
               v_cache=self.v_c[c], pos=self.pos)
        sparse_decode(self.q, self.k_c[c], self.v_c[c], self.lens, self.idx[c], out=self.out,
                      workspace=self.ws, params=self.p)
        self.io.send(q_t)                              # pack(t) -> the Cache Rank
        self.io.send(kv_t)
        self.packs += 1
        if self.rx is not None:
            self.rx.expect_one()                       # sel(t + 1) will answer it
        return self.out

    def finish(self) -> None:
        """Drain: take every selection the Cache Rank sent -- one per pack plus
        the first -- so no send is left waiting on the Cache Rank's side (with
        'reuse' some were skipped during the steps)."""
        while self.received < self.packs + 1:
            self._install()
        if self.rx is not None:
            self.rx.close()

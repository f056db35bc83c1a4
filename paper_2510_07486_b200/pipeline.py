"""a5 -- asynchronous selection: step t+1's token selection on a side stream,
overlapped with step t's attention and the rest of the layer.

The paper moves query prediction and top-k selection off the inference
critical path: once q_t is enqueued into the sliding window, the
selection for the NEXT step runs concurrently with the current step's work,
and the next step's attention only waits for its result (P:184-191,
P:262-268, Fig. 4).  On one GPU this becomes two CUDA streams:

    main  : [wait sel(t)] push q_t, k_t, v_t -> sparse_decode(idx[t%2]) -> forward
    side  :                    \\-> predict -> score_select -> idx[(t+1)%2] -> sel(t+1)

* idx is double-buffered by step parity.  The side stream writes
  idx[(t+1)%2] only after the push of step t, which main enqueues after
  decode(t-1) -- the last reader of that buffer -- so the write-after-read is
  ordered by the push event.
* Main waits for sel(t) before pushing step t's inputs: that both supplies
  step t's indices and guarantees the side stream has finished reading the
  window slot and the KV row that the push overwrites.
* Decode runs with n_fresh = 1: the newest token (whose K/V arrive after the
  selection was made) is always attended (reading R12).

Every compute step is a library kernel (predict_query, score_select,
sparse_decode; the synthetic forward is libasp_synth's weight-streaming
kernel); this module only orders them with torch streams and events.
"""
from __future__ import annotations

import torch

from . import predict_query, score_select, sparse_decode
from . import synth
from .step import DecodeStep


class AsyncPipeline:
    def __init__(self, step: DecodeStep, forward_bytes: int = 0, priority: str = "none"):
        if step.n_fresh != 1:
            raise ValueError("the async pipeline decodes with n_fresh = 1 (reading R12)")
        self.step = step
        dev = step.device
        # stream priorities (CTA scheduling order when both streams have work
        # pending): "none" (default, measured best overall), "main" (the step's
        # push / decode / forward first) or "side" (the selection chain first)
        if priority not in ("none", "main", "side"):
            raise ValueError("priority: none, main or side")
        top = torch.cuda.Stream.priority_range()[1] if priority != "none" else 0
        self.hi = (torch.cuda.Stream(device=dev, priority=top) if priority == "main" else None)
        self.side = torch.cuda.Stream(device=dev, priority=top if priority == "side" else 0)
        self.idx = [step.sel_idx, torch.empty_like(step.sel_idx)]
        self.ev_push = torch.cuda.Event()
        self.ev_sel = [torch.cuda.Event(), torch.cuda.Event()]
        self.weights = (torch.zeros(forward_bytes, dtype=torch.uint8, device=dev)
                        if forward_bytes > 0 else None)
        self.sink = torch.zeros(1, dtype=torch.float32, device=dev)
        # the fresh token's K/V land at seq_lens[b] - 1: lengths are held fixed
        # (the steady state), so the newest slot is overwritten each step and
        # decode's n_fresh = 1 tail attends exactly the pushed row
        self.pos = torch.empty_like(step.seq_lens)
        self.set_seq_lens(None)
        self.t = 0
        self.primed = False

    def set_seq_lens(self, lens) -> None:
        """Set the step's sequence lengths (None: keep them) and the push
        position seq_lens - 1 that goes with them (plumbing, not per step)."""
        s = self.step
        if lens is not None:
            s.seq_lens.copy_(torch.as_tensor(lens, dtype=torch.int32))
        torch.sub(s.seq_lens, 1, out=self.pos)

    # ------------------------------------------------------------------ pieces
    def select(self, buf: int, stream) -> None:
        """a1 -> a2+a3 into idx[buf] on `stream`."""
        s = self.step
        predict_query(s.window, s.q_hat, dev_flags=s.dev_flags, stream=stream, params=s.p_pred)
        score_select(s.q_hat, s.k_cache, s.seq_lens, s.cfg.top_k, sel_idx=self.idx[buf],
                     workspace=s.ws_sel, dev_flags=s.dev_flags, stream=stream, params=s.p_sel)

    def decode(self, buf: int, stream) -> None:
        s = self.step
        sparse_decode(s.q, s.k_cache, s.v_cache, s.seq_lens, self.idx[buf], out=s.out,
                      workspace=s.ws_dec, stream=stream, params=s.p_dec)

    def forward(self, stream) -> None:
        if self.weights is not None:
            synth.synthetic_forward(self.weights, self.sink, stream)

    def push(self, q_t=None, kv_t=None) -> None:
        """a0 on the current stream, one kernel (asyncspade_append): q_t into the
        window ring and (bf16) the current query, the new token's K/V rows into
        the newest cache slot (seq_lens[b] - 1; lengths are held fixed)."""
        s = self.step
        if q_t is not None:
            if kv_t is not None:
                s.append(q_t, kv_t[0], kv_t[1], self.pos)
            else:
                s.append(q_t)

    # ------------------------------------------------------------------ pipelined
    def prime(self) -> None:
        """Selection for the first step, on the side stream."""
        main = torch.cuda.current_stream(self.step.device)
        self.ev_push.record(main)
        self.side.wait_event(self.ev_push)
        self.select(self.t % 2, self.side)
        self.ev_sel[self.t % 2].record(self.side)
        self.primed = True

    def run_step(self, q_t=None, kv_t=None) -> None:
        """One decode step t, selection for t+1 overlapped."""
        if not self.primed:
            self.prime()
        caller = torch.cuda.current_stream(self.step.device)
        main = self.hi if self.hi is not None else caller
        if main is not caller:
            main.wait_stream(caller)              # the step's inputs come from the caller
        cur, nxt = self.t % 2, (self.t + 1) % 2
        main.wait_event(self.ev_sel[cur])
        with torch.cuda.stream(main):
            self.push(q_t, kv_t)
        self.ev_push.record(main)
        self.side.wait_event(self.ev_push)
        self.select(nxt, self.side)
        self.ev_sel[nxt].record(self.side)
        self.decode(cur, main)
        self.forward(main)
        if main is not caller:
            caller.wait_stream(main)              # outputs in the caller's order
        self.t += 1

    def drain(self) -> None:
        """Join the side stream into the current stream."""
        torch.cuda.current_stream(self.step.device).wait_stream(self.side)

    # ------------------------------------------------------------------ serial
    def run_step_serial(self, q_t=None, kv_t=None) -> None:
        """The same step with no overlap: decode(t) on idx selected before it,
        then select(t+1), all on the current stream (bit-identical results)."""
        main = torch.cuda.current_stream(self.step.device)
        cur, nxt = self.t % 2, (self.t + 1) % 2
        if not self.primed:
            self.select(cur, main)
            self.primed = True
        self.push(q_t, kv_t)
        self.select(nxt, main)
        self.decode(cur, main)
        self.forward(main)
        self.t += 1

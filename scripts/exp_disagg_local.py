"""Both disaggregated ranks in one process with an in-memory transport: does
the protocol reproduce the single-rank serial pipeline (isolates the kernels
and bookkeeping from the distributed transport)?"""
import os, sys, collections, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_07486_b200 import configs
from paper_2510_07486_b200.step import DecodeStep
from paper_2510_07486_b200.pipeline import AsyncPipeline
from paper_2510_07486_b200.disagg import CacheRank, InferenceRank

class Q:
    def __init__(self, inbox, outbox): self.inbox, self.outbox = inbox, outbox
    def send(self, t): self.outbox.append(t.clone())
    def recv(self, t): t.copy_(self.inbox.popleft())

cfg = configs.QWEN3_8B.with_(batch=2, seq_len=1024, top_k=128)
steps = 3
g = torch.Generator().manual_seed(11)
q_ts = [torch.randn(2, 32, 128, generator=g) for _ in range(steps)]
kvs = [torch.randn(2, 2, 8, 128, generator=g).to(torch.bfloat16) for _ in range(steps)]
st = DecodeStep(cfg, "cuda", n_fresh=1); st.fill_synthetic()
pipe = AsyncPipeline(st)
ref, ref_idx = [], []
for t in range(steps):
    cur = t % 2
    pipe.run_step_serial(q_ts[t].cuda(), kvs[t].cuda())
    ref.append(st.out.clone()); ref_idx.append(pipe.idx[cur].clone())
a, b = collections.deque(), collections.deque()
cr = CacheRank(cfg, "cuda", Q(a, b)); cr.step.fill_synthetic()
ir = InferenceRank(cfg, "cuda", Q(b, a), 32, 8, 2)
cr.prime()
for t in range(steps):
    o = ir.step(q_ts[t].cuda(), kvs[t].cuda()).clone()
    cr.serve(send=t < steps - 1)
    print(t, "out equal", torch.equal(o, ref[t]), "max diff", (o - ref[t]).abs().max().item(),
          "live entries", int((ir.idx >= 0).sum()), "ref valid", int(((ref_idx[t] >= 0) & (ref_idx[t] < 1023)).sum()))

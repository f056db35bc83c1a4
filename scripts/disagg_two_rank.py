"""Two-process (gloo, one GPU) disaggregation vs the single-rank serial a5
pipeline, per step (run by tests/test_gpu_parity.py; prints one line per step)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch.multiprocessing as mp
from paper_2510_07486_b200 import configs

def worker(rank, cfg, steps, q_np, kv_np, outq):
    # inputs and results cross the process boundary as numpy (pickled by value:
    # torch's shared-memory tensor passing races with the workers' exit)
    sys.path.insert(0, ROOT)
    q_ts = [torch.from_numpy(a) for a in q_np]
    kvs = [torch.from_numpy(a).view(torch.bfloat16) for a in kv_np]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29600 + os.getppid() % 500))
    import torch.distributed as dist
    from paper_2510_07486_b200.disagg import CacheRank, InferenceRank, Transport
    dist.init_process_group("gloo", rank=rank, world_size=2)
    io = Transport(1 - rank)
    if rank == 1:
        cr = CacheRank(cfg, "cuda", io); cr.step.fill_synthetic(); cr.prime()
        sels = [cr.i_sel.cpu().clone()]
        for t in range(steps):
            cr.serve(send=t < steps - 1); sels.append(cr.step.sel_idx.cpu().clone())
        outq.put(("cache", torch.stack(sels).numpy()))
    else:
        ir = InferenceRank(cfg, "cuda", io, 32, 8, 2)
        outs, idxs, ks = [], [], []
        for t in range(steps):
            outs.append(ir.step(q_ts[t].cuda(), kvs[t].cuda()).cpu().clone())
            idxs.append(ir.idx.cpu().clone()); ks.append(ir.k_c.cpu().clone())
        outq.put(("inf", (torch.stack(outs).numpy(), torch.stack(idxs).numpy(),
                          torch.stack(ks).view(torch.int16).numpy())))
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    from paper_2510_07486_b200.step import DecodeStep
    from paper_2510_07486_b200.pipeline import AsyncPipeline
    cfg = configs.QWEN3_8B.with_(batch=2, seq_len=1024, top_k=128)
    steps = 3
    g = torch.Generator().manual_seed(11)
    q_ts = [torch.randn(2, 32, 128, generator=g) for _ in range(steps)]
    kvs = [torch.randn(2, 2, 8, 128, generator=g).to(torch.bfloat16) for _ in range(steps)]
    st = DecodeStep(cfg, "cuda", n_fresh=1); st.fill_synthetic(); pipe = AsyncPipeline(st)
    ref, ref_idx = [], []
    for t in range(steps):
        pipe.run_step_serial(q_ts[t].cuda(), kvs[t].cuda()); ref.append(st.out.cpu().clone()); ref_idx.append(pipe.idx[t % 2].cpu().clone())
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    q_np = [t.numpy() for t in q_ts]
    kv_np = [t.view(torch.int16).numpy() for t in kvs]
    ps = [ctx.Process(target=worker, args=(r, cfg, steps, q_np, kv_np, q)) for r in range(2)]
    [p.start() for p in ps]
    res = dict(q.get(timeout=200) for _ in range(2))
    [p.join() for p in ps]
    outs, idxs, ks = res["inf"]
    outs, idxs = torch.from_numpy(outs), torch.from_numpy(idxs)
    ks = torch.from_numpy(ks).view(torch.bfloat16)
    for t in range(steps):
        live_ref = torch.where((ref_idx[t] >= 0) & (ref_idx[t] < 1023), torch.arange(128, dtype=torch.int32), torch.tensor(-1, dtype=torch.int32))
        print(t, "out eq", torch.equal(outs[t], ref[t]), "idx eq", torch.equal(idxs[t], live_ref),
              "fresh k eq", torch.equal(ks[t][:, :, 128], kvs[t][0]))

"""Two-process dual-rank run: an Inference Rank and a
Cache Rank (paper_2510_07486_b200/disagg.py) exchange packs and selections for
T steps; rank 0 writes what happened to an .npz for the caller to check:

    outs   [T, B, Hq, D] fp32   Inference Rank outputs
    used   [T]                  which selection (0 = the prime) each step used
    sent   [T + 1, B, Hkv, k]   the Cache Rank's global selections, in order
    q_ts   [T, B, Hq, D] fp32, kvs [T, 2, B, Hkv, D] bf16 bits: the step inputs

usage: disagg_two_rank.py OUT.npz [--backend gloo|nccl] [--policy wait|reuse]
                                  [--late STEP] [--steps T] [--reference]
gloo: both ranks on cuda:0 (tests); nccl: rank r on cuda:r (a 2-GPU node),
which also prints per-step timings (the paper's Table 3 quantities on B200:
Inference-Rank step latency and Cache-Rank per-step management latency).
--reference: also run the single-rank serial a5 pipeline on the same inputs
(wait policy: the outputs must match bit for bit) into the same .npz.
"""
import argparse
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2510_07486_b200 import configs  # noqa: E402

CFG = configs.QWEN3_8B.with_(batch=2, seq_len=1024, top_k=128)


def _inputs(cfg, steps):
    g = torch.Generator().manual_seed(11)
    q_ts = [torch.randn(cfg.batch, cfg.n_q_heads, cfg.head_dim, generator=g) for _ in range(steps)]
    kvs = [torch.randn(2, cfg.batch, cfg.n_kv_heads, cfg.head_dim, generator=g).to(torch.bfloat16)
           for _ in range(steps)]
    return q_ts, kvs


def worker(rank, args, port, outq):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2510_07486_b200.disagg import CacheRank, InferenceRank, Transport
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank if args.backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    dist.init_process_group(args.backend, rank=rank, world_size=2,
                            **({"device_id": dev} if args.backend == "nccl" else {}))
    g_pack = dist.new_group([0, 1])               # inference -> cache
    g_sel = dist.new_group([0, 1])                # cache -> inference
    cfg, T = CFG, args.steps
    q_ts, kvs = _inputs(cfg, T)
    if rank == 1:                                  # Cache Rank
        cr = CacheRank(cfg, dev, Transport(0, g_sel, g_pack))
        cr.step.fill_synthetic()
        torch.cuda.synchronize()
        cr.prime(keep=True)
        t_serve = []
        for t in range(T):
            t0 = time.perf_counter()
            cr.serve(keep=True, delay_s=0.5 if t == args.late else 0.0)
            torch.cuda.synchronize()
            t_serve.append(time.perf_counter() - t0)
        outq.put(("cache", (np.stack([s.numpy() for s in cr.sent]), t_serve)))
    else:                                          # Inference Rank
        ir = InferenceRank(cfg, dev, Transport(1, g_pack, g_sel), cfg.n_q_heads,
                           cfg.n_kv_heads, cfg.batch, stall_policy=args.policy)
        outs, t_step = [], []
        for t in range(T):
            qd, kd = q_ts[t].to(dev), kvs[t].to(dev)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            o = ir.step(qd, kd)
            torch.cuda.synchronize()
            t_step.append(time.perf_counter() - t0)
            outs.append(o.cpu().clone())
            if args.policy == "reuse" and t == args.late:
                time.sleep(0.05)                   # let the late selection land meanwhile
        ir.finish()
        outq.put(("inf", (torch.stack(outs).numpy(), np.array(ir.used), t_step)))
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--backend", default="gloo", choices=["gloo", "nccl"])
    ap.add_argument("--policy", default="wait", choices=["wait", "reuse"])
    ap.add_argument("--late", type=int, default=-1, help="Cache-Rank step that sends late")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--reference", action="store_true")
    args = ap.parse_args()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, args, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    outs, used, t_step = res["inf"]
    sent, t_serve = res["cache"]
    q_ts, kvs = _inputs(CFG, args.steps)
    extra = {}
    if args.reference:
        from paper_2510_07486_b200.pipeline import AsyncPipeline
        from paper_2510_07486_b200.step import DecodeStep
        st = DecodeStep(CFG, "cuda", n_fresh=1)
        st.fill_synthetic()
        pipe = AsyncPipeline(st)
        ref = []
        for t in range(args.steps):
            pipe.run_step_serial(q_ts[t].cuda(), kvs[t].cuda())
            ref.append(st.out.cpu().clone())
        extra["ref_outs"] = torch.stack(ref).numpy()
    np.savez(args.out, outs=outs, used=used, sent=sent,
             q_ts=torch.stack(q_ts).numpy(),
             kvs=torch.stack(kvs).view(torch.int16).numpy().view(np.uint16), **extra)
    print(f"backend {args.backend} policy {args.policy} late {args.late}: used {used.tolist()}; "
          f"inference step ms {[round(x * 1e3, 3) for x in t_step]}; "
          f"cache serve ms {[round(x * 1e3, 3) for x in t_serve]}")


if __name__ == "__main__":
    main()

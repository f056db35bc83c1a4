"""Sweeps of BASELINE.json configs [3] and [4] on one B200.
Steps are replayed from a CUDA graph (the per-call host cost would otherwise
bound the small ones).

    python scripts/sweep.py long-cot          # [3] batch 8, ctx 4k..512k, per-GPU shard of P = 8
    python scripts/sweep.py high-concurrency  # [4] Qwen3-8B shape, ctx 4k, batch 1..512, a5 overlap
    python scripts/sweep.py layer-packed      # NEXT-2: P_l layers per launch (small shapes)
    python scripts/sweep.py quest             # NEXT-4: Quest page-bound comparator vs AsyncSpade

One JSON line per point.  Times are CUDA events on the launching stream over
`--steps` back-to-back steps after `--warmup`, per step in µs.  Core bytes as
in bench.py (full-K read + selected K and V).  For [4] the a5 overlap is
measured with the synthetic forward (a 386 MB weight-streaming read, Qwen3-8B
layer parameters) on the main stream:
  t_fwd        forward alone
  t_sel        a1 predict + a2/a3 score_select alone
  t_dec        a4 sparse decode alone
  t_serial     push + select + decode + forward on one stream
  t_overlapped the AsyncPipeline step (selection for t+1 on a side stream)
  overlap_eff  (t_serial - t_overlapped) / min(t_fwd, t_sel)
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_07486_b200 as asp  # noqa: E402
from paper_2510_07486_b200 import configs, synth  # noqa: E402
from paper_2510_07486_b200.pipeline import AsyncPipeline  # noqa: E402
from paper_2510_07486_b200.step import DecodeStep  # noqa: E402


def _peak():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        return float(json.load(f)["hbm_gbs"])


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3                   # µs per step


def point(cfg, args, kv_heads=None, overlap=False):
    step = DecodeStep(cfg, "cuda", kv_heads=kv_heads, n_fresh=1 if overlap else 0)
    step.fill_synthetic()
    torch.cuda.synchronize()
    hn = step.n_kv
    core = cfg.core_bytes(hn)
    # CUDA-graph replay (PDL edges kept): small steps are otherwise bound by the
    # host's per-call launch cost, not the GPU
    step.capture()
    t_step = timed(step.replay, args.steps, args.warmup)
    res = {"workload": cfg.name, "batch": cfg.batch, "seq_len": cfg.seq_len, "top_k": cfg.top_k,
           "kv_heads_on_gpu": hn, "us_per_step": t_step,
           "hbm_tb_per_s": core / (t_step * 1e-6) / 1e12,
           "roofline_frac": core / (t_step * 1e-6) / 1e9 / _peak(), "core_bytes": core}
    if overlap:
        pipe = AsyncPipeline(step, forward_bytes=2 * synth.QWEN3_8B_LAYER_PARAMS)
        main = torch.cuda.current_stream()
        B, D = cfg.batch, cfg.head_dim
        q_t = torch.randn(B, step.n_q, D, device="cuda")
        kv_t = torch.randn(2, B, hn, D, device="cuda").to(torch.bfloat16)
        res["t_fwd"] = timed(lambda: pipe.forward(main), args.steps, args.warmup)
        res["t_sel"] = timed(lambda: pipe.select(0, main), args.steps, args.warmup)
        res["t_dec"] = timed(lambda: pipe.decode(0, main), args.steps, args.warmup)
        res["t_serial"] = timed(lambda: pipe.run_step_serial(q_t, kv_t), args.steps, args.warmup)

        def overlapped():
            pipe.run_step(q_t, kv_t)

        for _ in range(args.warmup):
            overlapped()
        pipe.drain()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            overlapped()
        pipe.drain()
        e1.record()
        torch.cuda.synchronize()
        res["t_overlapped"] = e0.elapsed_time(e1) / args.steps * 1e3
        res["overlap_eff"] = ((res["t_serial"] - res["t_overlapped"]) /
                              min(res["t_fwd"], res["t_sel"]))
        res["forward_bytes"] = 2 * synth.QWEN3_8B_LAYER_PARAMS
    del step
    torch.cuda.empty_cache()
    return res


def quest_point(cfg, args, P=16):
    step = DecodeStep(cfg, "cuda")
    step.fill_synthetic()
    torch.cuda.synchronize()
    B, Hkv, L, D, k = cfg.batch, cfg.n_kv_heads, cfg.seq_len, cfg.head_dim, cfg.top_k
    q32 = step.q.float()
    meta = asp.quest_summarize(step.k_cache, step.seq_lens, P, k, cfg.n_q_heads)
    ws = torch.empty(max(int(asp.lib().asyncspade_quest_select_workspace(
        ctypes.byref(asp.SelectParams(B, cfg.n_q_heads, Hkv, D, k, L, 0,
                                      *step.k_cache.stride()[:3])), P)), 256),
                     dtype=torch.uint8, device="cuda")
    idx_q = torch.empty_like(step.sel_idx)

    def quest_step():
        asp.quest_select(q32, meta, step.k_cache, step.seq_lens, k, P, sel_idx=idx_q,
                         workspace=ws)
        asp.sparse_decode(step.q, step.k_cache, step.v_cache, step.seq_lens, idx_q, out=step.out,
                          workspace=step.ws_dec, params=step.p_dec)

    t_asp = timed(step.run, args.steps, args.warmup)
    t_quest = timed(quest_step, args.steps, args.warmup)
    t_qsel = timed(lambda: asp.quest_select(q32, meta, step.k_cache, step.seq_lens, k, P,
                                            sel_idx=idx_q, workspace=ws), args.steps, args.warmup)
    t_sum = timed(lambda: asp.quest_summarize(step.k_cache, step.seq_lens, P, k, cfg.n_q_heads,
                                              meta=meta), 3, 1)
    # selection quality: overlap with the exact token top-k of the current query
    step.run()
    exact = asp.score_select(q32, step.k_cache, step.seq_lens, k)
    quest_step()
    torch.cuda.synchronize()

    def overlap(a):
        n = 0
        ea, eb = a.view(-1, k).cpu(), exact.view(-1, k).cpu()
        for r in range(ea.shape[0]):
            n += len(set(ea[r].tolist()) & set(eb[r].tolist()))
        return n / (ea.shape[0] * k)

    meta_bytes = B * Hkv * ((L + P - 1) // P) * 2 * D * 2
    kv_sel = 2 * B * Hkv * k * D * 2
    res = {"workload": cfg.name, "page_size": P, "asyncspade_step_us": t_asp,
           "quest_step_us": t_quest, "quest_select_us": t_qsel, "quest_summarize_us": t_sum,
           "quest_bytes_per_step": meta_bytes + kv_sel,
           "asyncspade_bytes_per_step": cfg.core_bytes(),
           "quest_select_tb_per_s": meta_bytes / (t_qsel * 1e-6) / 1e12,
           "overlap_with_exact_topk": {"asyncspade_predicted_query": overlap(step.sel_idx),
                                       "quest_current_query": overlap(idx_q)},
           "note": "Quest runs on the critical path (current query); AsyncSpade's selection "
                   "can run a step ahead (a5); synthetic N(0,1) keys, AR(1) queries"}
    del step
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweep", choices=["long-cot", "high-concurrency", "layer-packed", "quest",
                                      "gather", "groups", "table3"])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default="", help="comma list of batch sizes (high-concurrency) "
                    "or log2 contexts (long-cot) to run")
    args = ap.parse_args()
    only = {int(x) for x in args.only.split(",") if x}
    asp.lib()
    lines = []
    if args.sweep == "long-cot":
        for e in range(12, 20):                                # 4k .. 512k
            if only and e not in only:
                continue
            cfg = configs.long_cot(1 << e)
            lines.append(point(cfg, args, kv_heads=(0, 1)))     # per-GPU shard at P = 8
            print(json.dumps(lines[-1]), flush=True)
    elif args.sweep == "quest":
        # NEXT-4 comparator: Quest selects
        # pages of 16 by an upper bound with the CURRENT query (critical path);
        # AsyncSpade selects tokens with the predicted query.  Step times and the
        # overlap ratio (Eq. 1) of each selection with the exact
        # token top-k of the current query.
        for cfg in (configs.QWEN3_8B, configs.QWEN3_32B):
            lines.append(quest_point(cfg, args))
            print(json.dumps(lines[-1]), flush=True)
    elif args.sweep == "groups":
        # GQA group size 1..32 at a fixed KV cache (B = 16, 8 KV heads, 32k, k = 2048): the
        # score stream stays HBM-bound as G (the contraction's intensity) grows
        for G in (1, 2, 4, 8, 16, 32):
            cfg = configs.Config(f"groups_g{G}_b16_ctx32k", 2, 16, 8 * G, 8, 128, 32768, 2048, 16)
            lines.append(point(cfg, args))
            lines[-1]["group"] = G
            print(json.dumps(lines[-1]), flush=True)
    elif args.sweep == "gather":
        # NEXT-1: the Cache Rank's payload (asyncspade_gather_filtered) per layer
        for cfg in (configs.QWEN3_8B, configs.QWEN3_32B, configs.high_concurrency(8)):
            step = DecodeStep(cfg, "cuda")
            step.fill_synthetic()
            step.run()
            ko = torch.empty(cfg.batch, cfg.n_kv_heads, cfg.top_k, cfg.head_dim,
                             dtype=torch.bfloat16, device="cuda")
            vo, io = torch.empty_like(ko), torch.empty_like(step.sel_idx)
            t = timed(lambda: asp.gather_filtered(step.k_cache, step.v_cache, step.seq_lens,
                                                  step.sel_idx, n_fresh=1, k_out=ko, v_out=vo,
                                                  idx_out=io), args.steps, args.warmup)
            payload = 2 * ko.numel() * 2 + io.numel() * 4
            lines.append({"workload": cfg.name, "gather_us": t, "payload_bytes": payload,
                          "gather_tb_per_s": 2 * payload / (t * 1e-6) / 1e12,
                          "nvlink_900GBps_us": payload / 900e9 * 1e6})
            print(json.dumps(lines[-1]), flush=True)
            del step
            torch.cuda.empty_cache()
    elif args.sweep == "table3":
        # NEXT-1, the paper's Table 3 on one B200: per pack of P_l
        # layers, the Cache Rank's management latency (append the pack, predict,
        # score + top-k, gather the selected rows into the receiver's layout --
        # our kernels, layer-packed, CUDA-graph replay), an Inference-Rank proxy
        # (the pack's weight streaming -- a batch-8/16 decode forward is bound by
        # reading the layers' bf16 weights -- plus the sparse decode over the
        # compact cache), and the minimal link bandwidth for full overlap =
        # bytes exchanged per pack / inference time (the NVLink transfer itself
        # needs two GPUs and is not measured).  Paper's H100 rows for context.
        rows = [("qwen3-8b", 8, 32768, 2048, (6, 12), (5.47, 3.92, 140.40)),
                ("qwen3-8b", 16, 16384, 1024, (6, 12), (5.91, 5.18, 129.94)),
                ("qwen3-32b", 8, 32768, 2048, (4, 8), (4.39, 3.74, 228.88)),
                ("qwen3-32b", 16, 16384, 1024, (4, 8), (4.37, 3.72, 229.93))]
        for model, B, L, k, packs, h100 in rows:
            base = configs.QWEN3_8B if model == "qwen3-8b" else configs.QWEN3_32B
            cfg = base.with_(batch=B, seq_len=L, top_k=k)
            layer_params = (synth.QWEN3_8B_LAYER_PARAMS if model == "qwen3-8b"
                            else synth.QWEN3_32B_LAYER_PARAMS)
            for pl in packs:
                st = DecodeStep(cfg, "cuda", layers=pl, n_fresh=1)
                st.fill_synthetic()
                Bp, D = B * pl, cfg.head_dim
                g = torch.Generator(device="cpu").manual_seed(3)
                q_t = torch.randn(Bp, st.n_q, D, generator=g).cuda()
                kv_t = torch.randn(2, Bp, st.n_kv, D, generator=g).to(torch.bfloat16).cuda()
                pos = st.seq_lens - 1
                k_sel = torch.empty(Bp, st.n_kv, k + 1, D, dtype=torch.bfloat16, device="cuda")
                v_sel = torch.empty_like(k_sel)
                i_sel = torch.empty(Bp, st.n_kv, k, dtype=torch.int32, device="cuda")

                def cache_mgmt():
                    # the pack arrives (ring position fixed: the timing is per pack)
                    asp.append(q_t, st.window, 0, q_cur=st.q, k_new=kv_t[0], v_new=kv_t[1],
                               k_cache=st.k_cache, v_cache=st.v_cache, pos=pos)
                    asp.predict_query(st.window, st.q_hat, params=st.p_pred)
                    asp.score_select(st.q_hat, st.k_cache, st.seq_lens, k, sel_idx=st.sel_idx,
                                     workspace=st.ws_sel, params=st.p_sel)
                    asp.gather_filtered(st.k_cache, st.v_cache, st.seq_lens, st.sel_idx,
                                        n_fresh=1, k_out=k_sel[:, :, :k], v_out=v_sel[:, :, :k],
                                        idx_out=i_sel)
                t_cache = timed(cache_mgmt, args.steps, args.warmup)
                del st
                torch.cuda.empty_cache()
                weights = torch.zeros(2 * layer_params * pl, dtype=torch.uint8, device="cuda")
                sink = torch.zeros(1, dtype=torch.float32, device="cuda")
                t_fwd = timed(lambda: synth.synthetic_forward(weights, sink), args.steps, args.warmup)
                del weights
                q_b = torch.zeros(Bp, cfg.n_q_heads, D, dtype=torch.bfloat16, device="cuda")
                lens = torch.full((Bp,), k + 1, dtype=torch.int32, device="cuda")
                pd = asp.decode_params(q_b, k_sel, v_sel, k, 1)
                ws = torch.zeros(asp.sparse_decode_workspace(pd), dtype=torch.uint8, device="cuda")
                out = torch.empty(Bp, cfg.n_q_heads, D, dtype=torch.float32, device="cuda")
                t_attn = timed(lambda: asp.sparse_decode(q_b, k_sel, v_sel, lens, i_sel, out=out,
                                                         workspace=ws, params=pd),
                               args.steps, args.warmup)
                payload = (k_sel.numel() + v_sel.numel()) * 2 + i_sel.numel() * 4 \
                    + q_t.numel() * 4 + kv_t.numel() * 2
                t_inf = t_fwd + t_attn
                lines.append({"workload": f"{model} B{B} {L // 1024}k select {k // 1024}k",
                              "packed_layers": pl, "cache_management_ms": t_cache / 1e3,
                              "inference_proxy_ms": t_inf / 1e3, "forward_weights_ms": t_fwd / 1e3,
                              "sparse_attention_ms": t_attn / 1e3,
                              "payload_bytes_per_pack": payload,
                              "minimal_bandwidth_GBps": payload / (t_inf * 1e-6) / 1e9,
                              "overlapped": t_cache <= t_inf,
                              "paper_h100_inference_ms_cache_ms_GBps": h100})
                print(json.dumps(lines[-1]), flush=True)
                del k_sel, v_sel, i_sel, q_b, out, ws
                torch.cuda.empty_cache()
    elif args.sweep == "layer-packed":
        # NEXT-2: per-layer step time when P_l layers share one
        # launch of each kernel, on the small shapes that under-fill the SMs
        for cfg, kvh in [(configs.high_concurrency(1), None), (configs.high_concurrency(8), None),
                         (configs.high_concurrency(32), None), (configs.QWEN3_32B, (0, 1))]:
            for pl in (1, 2, 4, 8):
                step = DecodeStep(cfg, "cuda", kv_heads=kvh, layers=pl)
                step.fill_synthetic()
                step.capture()
                t = timed(step.replay, args.steps, args.warmup)
                core = cfg.core_bytes(step.n_kv) * pl
                lines.append({"workload": cfg.name, "kv_heads_on_gpu": step.n_kv, "layers_packed": pl,
                              "us_per_launch": t, "us_per_layer": t / pl,
                              "hbm_tb_per_s": core / (t * 1e-6) / 1e12,
                              "roofline_frac": core / (t * 1e-6) / 1e9 / _peak()})
                print(json.dumps(lines[-1]), flush=True)
                del step
                torch.cuda.empty_cache()
    else:
        for e in range(0, 10):                                 # batch 1 .. 512
            if only and (1 << e) not in only:
                continue
            cfg = configs.high_concurrency(1 << e)
            lines.append(point(cfg, args, overlap=True))
            print(json.dumps(lines[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for ln in lines:
                f.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()

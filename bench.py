#!/usr/bin/env python
"""bench.py -- AsyncSpade decode hot path on B200 (one attention layer's step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl asyncspade|reference]

Workload: BASELINE.json configs[2] -- Qwen3-32B attention shape (64 q heads /
8 KV heads, head_dim 128), batch 64, 32k context, top-k 2048 (1/16), window 16
-- with seeded synthetic inputs.  A step is one pass of the
whole path: a1 predict -> a2 score -> a3 top-k -> a4 sparse decode (SURVEY
§8(a)).  N > 1 (torchrun, one rank per GPU): KV heads are sharded over ranks
(total work fixed -> "strong" scaling), no collective inside the step; the
output all-gather (NCCL) is timed separately.

Prints ONE JSON line (rank 0).  Timing: device CUDA events on the launching
stream, W warm-up steps, barrier + synchronize around exactly K steps, max
over ranks.  Inputs (K + V = 8.6 GB at N = 1) are far larger than the 126 MB
L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "µs/decode step (select+sparse attn) & HBM TB/s, Qwen3-32B bs64 ctx32k"
UNIT = "us/step"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="asyncspade", choices=["asyncspade", "reference"])
    ap.add_argument("--config", default="qwen3-32b_b64_ctx32k")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-a5", action="store_true",
                    help="skip the a5 (asynchronous selection) pipelined measurement")
    ap.add_argument("--a5-no-forward", action="store_true",
                    help="a5 without the layer's synthetic forward (the step alone)")
    ap.add_argument("--a5-priority", default="none", choices=["none", "main", "side"])
    ap.add_argument("--emulate-shard", type=int, default=0, metavar="P",
                    help="one GPU runs rank 0's shard of a P-way KV-head split (the per-GPU "
                         "work of the P-GPU run; scaling evidence when only one GPU is at hand)")
    ap.add_argument("--bf16-window", action="store_true",
                    help="keep the query window ring in bf16 (ASP_WINDOW_BF16)")
    ap.add_argument("--ragged", action="store_true",
                    help="ragged batch: seq_lens seeded-uniform in [L/8, L] (the cache capacity "
                         "stays L; headline bytes count each row's own length)")
    ap.add_argument("--paged", type=int, default=0, metavar="PAGE_SIZE",
                    help="run on a paged KV pool (HND pages of PAGE_SIZE tokens, random page "
                         "placement) through the *_paged entry points (SURVEY §8(f) NEXT-4)")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: skip clocks, e2e and the CPU baseline")
    ap.add_argument("--eager", action="store_true",
                    help="time eager back-to-back launches instead of CUDA-graph replays")
    ap.add_argument("--launch-check", action="store_true",
                    help="multi-rank plumbing only (no kernels; gloo on CPU): every rank "
                         "reports its shard, rank 0 prints one JSON line")
    return ap.parse_args()


def _self_launch(args) -> None:
    """`bench.py --gpus N` (N > 1) outside torchrun: re-exec under
    torch.distributed.run with one rank per GPU (127.0.0.1 rendezvous)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def launch_check(args, cfg) -> None:
    """The multi-rank plumbing of the GPU arm without kernels: rendezvous,
    the §8(e) partition (shard_units), a MAX all-reduce of per-rank times and
    the head-major output gather, on gloo (CPU) or NCCL."""
    import torch
    import torch.distributed as dist
    from paper_2510_07486_b200 import shard as sh_mod
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo")
    sh = sh_mod.shard_units(cfg.batch, cfg.n_kv_heads, world, rank)
    q0, qn = sh.q_heads(cfg.group)
    # a stand-in output block: value = global (q head, batch) id, head-major
    hq = torch.arange(q0, q0 + qn, dtype=torch.float64)[:, None]
    bb = torch.arange(sh.b0, sh.b0 + sh.bn, dtype=torch.float64)[None, :]
    blk = (hq * cfg.batch + bb).contiguous()
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    if world > 1:
        full = sh_mod.gather_units(blk, sh, cfg.batch, cfg.n_q_heads, cfg.group)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        shards = [None] * world
        dist.all_gather_object(shards, [sh.b0, sh.bn, sh.h0, sh.hn])
    else:
        full, shards = blk, [[sh.b0, sh.bn, sh.h0, sh.hn]]
    ok = bool(torch.equal(full, torch.arange(cfg.n_q_heads * cfg.batch,
                                             dtype=torch.float64).view(cfg.n_q_heads, cfg.batch)))
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "config": cfg.name,
                          "shards_b0_bn_h0_hn": shards, "max_over_ranks": float(t[0]),
                          "gather_ok": ok}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic():
    """dram bytes per launch of the dominant call, from the committed ncu
    --set full summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("score_select_dram_bytes_per_launch")
    return None


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- reference arm
# The oracle as it stands (plain C, one thread per call), run on every host
# core at once: one worker process per core, each owning a few (batch,
# kv-head) rows whose inputs it generates BEFORE the timed region (generation
# is not the oracle).  A timed "round" = every worker runs the full oracle
# step (c1 -> c2 -> c3 -> c4) on one of its rows; its wall time is
# max(end) - min(start) over the workers (CLOCK_MONOTONIC, shared by the
# processes).  Scaled to the workload's row count.
def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_rows(cfg, rows, seed):
    """Host inputs for (b, kv-head) rows (generation excluded from timing)."""
    from paper_2510_07486_b200 import synth
    G, D, L = cfg.group, cfg.head_dim, cfg.seq_len
    data = []
    for r in rows:
        b, h = divmod(int(r), cfg.n_kv_heads)
        win, q = synth.query_trace(seed, cfg.batch, cfg.n_q_heads, cfg.window, D, b0=b,
                                   h0=h * G, batch_slice=1, head_slice=G)
        K = synth.kv_rows(seed, synth.STREAM_K, b, h, 0, L, cfg.n_kv_heads, L, D)[None, None]
        V = synth.kv_rows(seed, synth.STREAM_V, b, h, 0, L, cfg.n_kv_heads, L, D)[None, None]
        data.append((win, q, K, V))
    return data


def _oracle_worker(cfg_name, rows, seed, cmd_q, res_q):
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2510_07486_b200 import configs
    cfg = configs.by_name(cfg_name)
    data = _oracle_rows(cfg, rows, seed)
    oracle.build()
    res_q.put(("ready", None, None))
    while True:
        i = cmd_q.get()
        if i is None:
            return
        win, q, K, V = data[i % len(data)]
        t0 = time.perf_counter()
        oracle.step(win, q, K, V, [cfg.seq_len], cfg.top_k)
        res_q.put(("done", t0, time.perf_counter()))


class OraclePool:
    """One oracle worker process per host core (os.sched_getaffinity)."""

    def __init__(self, cfg, rows_per_worker: int, cores: int | None = None, seed=None):
        import multiprocessing as mp
        from paper_2510_07486_b200 import synth
        self.cfg = cfg
        self.cores = cores or len(os.sched_getaffinity(0))
        n_rows = cfg.batch * cfg.n_kv_heads
        seed = synth.base_seed(cfg.index) if seed is None else seed
        ctx = mp.get_context("spawn")
        self.res_q = ctx.Queue()
        self.cmd_qs, self.procs = [], []
        for w in range(self.cores):
            rows = [((w * rows_per_worker + j) * 37) % n_rows for j in range(rows_per_worker)]
            cq = ctx.Queue()
            pr = ctx.Process(target=_oracle_worker, args=(cfg.name, rows, seed, cq, self.res_q),
                             daemon=True)
            pr.start()
            self.cmd_qs.append(cq)
            self.procs.append(pr)
        for _ in range(self.cores):
            self.res_q.get(timeout=600)

    def round(self, i: int) -> float:
        """Every worker runs the full oracle step on its i-th row; wall seconds."""
        for cq in self.cmd_qs:
            cq.put(i)
        ts = [self.res_q.get(timeout=600) for _ in self.cmd_qs]
        return max(t[2] for t in ts) - min(t[1] for t in ts)

    def close(self):
        for cq in self.cmd_qs:
            cq.put(None)
        for pr in self.procs:
            pr.join(timeout=10)


def _single_thread_us_per_row(cfg, n_rows: int = 8) -> float:
    """One thread, the oracle's full step on a fixed n-row subset."""
    import oracle
    from paper_2510_07486_b200 import synth
    total = cfg.batch * cfg.n_kv_heads
    rows = [int(i * total / min(n_rows, total)) for i in range(min(n_rows, total))]
    data = _oracle_rows(cfg, rows, synth.base_seed(cfg.index))
    t0 = time.perf_counter()
    for win, q, K, V in data:
        oracle.step(win, q, K, V, [cfg.seq_len], cfg.top_k)
    return (time.perf_counter() - t0) / len(rows) * 1e6


def cpu_baseline(cfg, target_rounds: int = 4):
    """The oracle, as it stands, on all host cores: `target_rounds` rounds of
    one row per core (a bounded sample of the workload), scaled to a whole
    step; plus the one-thread time of configs [0] and [1] on 8 rows."""
    from paper_2510_07486_b200 import configs
    pool = OraclePool(cfg, rows_per_worker=target_rounds)
    try:
        pool.round(0)                                            # warm (page-in, caches)
        walls = [pool.round(i) for i in range(target_rounds)]
    finally:
        pool.close()
    rows_done = pool.cores * target_rounds
    n_rows_total = cfg.batch * cfg.n_kv_heads
    wall = sum(walls)
    us_per_step = wall / rows_done * n_rows_total * 1e6
    single = {c.name: _single_thread_us_per_row(c) * c.batch * c.n_kv_heads
              for c in (configs.TINY, configs.QWEN3_8B)}
    return {"value": us_per_step, "unit": UNIT, "cores": pool.cores, "kind": "oracle",
            "cpu_model": _cpu_model(),
            "sample": f"{rows_done} of {n_rows_total} (batch, kv-head) rows of {cfg.name} "
                      f"({target_rounds} rounds x {pool.cores} worker processes, one row each), "
                      f"full oracle step (fp64 predict, fp64 score, full sort, fp64 decode), "
                      f"scaled to a whole step; {wall:.2f} s wall",
            "single_thread_us_per_step": single,
            "single_thread_sample": "8 fixed rows (all rows of the tiny config), one thread, "
                                    "scaled to the config's whole step"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_rows_total = cfg.batch * cfg.n_kv_heads
    pool = OraclePool(cfg, rows_per_worker=4)
    try:
        for i in range(args.warmup):
            pool.round(i)
        per_row = []
        for i in range(args.steps):
            per_row.append(pool.round(i) / pool.cores)
    finally:
        pool.close()
    v = statistics.mean(per_row) * n_rows_total * 1e6
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": v / 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "batch": cfg.batch, "n_q_heads": cfg.n_q_heads,
                       "n_kv_heads": cfg.n_kv_heads, "head_dim": cfg.head_dim,
                       "seq_len": cfg.seq_len, "top_k": cfg.top_k, "window": cfg.window},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": pool.cores, "kind": "oracle",
                             "cpu_model": _cpu_model(),
                             "sample": f"per step: {pool.cores} of {n_rows_total} (batch, kv-head) "
                                       f"rows, one per core (worker process), full oracle step, "
                                       f"scaled to a whole step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def main():
    args = _args()
    from paper_2510_07486_b200 import configs
    cfg = configs.by_name(args.config)
    _self_launch(args)
    if args.launch_check:
        return launch_check(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    import paper_2510_07486_b200 as asp
    from paper_2510_07486_b200 import synth
    from paper_2510_07486_b200.step import DecodeStep

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_07486_b200.shard import shard_units
    shards = args.emulate_shard if (args.emulate_shard and world == 1) else world
    sh = shard_units(cfg.batch, cfg.n_kv_heads, shards, rank)   # §8(e): KV heads, then batch
    h0, hn = sh.h0, sh.hn
    wdt = torch.bfloat16 if args.bf16_window else torch.float32
    # multi-GPU: head-major outputs, so the gather below is one concatenation
    step = DecodeStep(cfg, "cuda", kv_heads=(h0, hn), window_dtype=wdt,
                      batch_range=(sh.b0, sh.bn), out_head_major=world > 1)
    step.fill_synthetic()
    lens = [cfg.seq_len] * sh.bn
    if args.ragged:
        import numpy as np
        rng = np.random.default_rng(synth.base_seed(cfg.index) + 99)
        lens = [int(x) for x in rng.integers(cfg.seq_len // 8, cfg.seq_len + 1, cfg.batch)]
        lens = lens[sh.b0:sh.b0 + sh.bn]
        step.seq_lens.copy_(torch.tensor(lens, dtype=torch.int32))
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)
    pool = None
    if args.paged:
        # the same logical cache scattered over a pool (random page placement)
        k_pool, bt = asp.page_pool(step.k_cache, args.paged, torch.Generator().manual_seed(7))
        step.k_cache = None
        torch.cuda.empty_cache()
        v_pool, _ = asp.page_pool(step.v_cache, args.paged, torch.Generator().manual_seed(7))
        step.v_cache = None
        torch.cuda.empty_cache()
        pool = (k_pool, v_pool, bt)
        args.no_e2e = args.no_a5 = True

    def one_step_paged(evs=None):
        k_pool, v_pool, bt = pool
        if evs is not None:
            evs[0].record(stream)
        asp.predict_query(step.window, step.q_hat, dev_flags=step.dev_flags, params=step.p_pred)
        if evs is not None:
            evs[1].record(stream)
        asp.score_select_paged(step.q_hat, k_pool, bt, step.seq_lens, cfg.top_k, cfg.seq_len,
                               sel_idx=step.sel_idx, workspace=step.ws_sel,
                               dev_flags=step.dev_flags)
        if evs is not None:
            evs[2].record(stream)
        asp.sparse_decode_paged(step.q, k_pool, v_pool, bt, step.seq_lens, step.sel_idx,
                                cfg.seq_len, out=step.out, workspace=step.ws_dec)
        if evs is not None:
            evs[3].record(stream)

    def one_step(evs=None, out=None):
        if pool is not None:
            return one_step_paged(evs)
        if evs is not None:
            evs[0].record(stream)
        asp.predict_query(step.window, step.q_hat, dev_flags=step.dev_flags, params=step.p_pred)
        if evs is not None:
            evs[1].record(stream)
        asp.score_select(step.q_hat, step.k_cache, step.seq_lens, cfg.top_k, sel_idx=step.sel_idx,
                         workspace=step.ws_sel, dev_flags=step.dev_flags, params=step.p_sel)
        if evs is not None:
            evs[2].record(stream)
        asp.sparse_decode(step.q, step.k_cache, step.v_cache, step.seq_lens, step.sel_idx,
                          out=step.out if out is None else out, workspace=step.ws_dec,
                          params=step.p_dec)
        if evs is not None:
            evs[3].record(stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 1)):
        one_step()
    barrier()
    # (1) the headline: K steps replayed from CUDA graphs; a
    #     graph holds `per_graph` consecutive steps, so the programmatic
    #     dependent launch edges between one step's last kernel and the next
    #     step's first are kept inside it; device events only around the
    #     whole region.  --eager: the same K steps as eager launches.
    per_graph = 1 if args.eager else min(10, args.steps)
    graphs = {}

    def graph_of(n):
        if n not in graphs:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                one_step()                       # warm the side stream's first launch
            stream.wait_stream(side)
            with torch.cuda.graph(g):
                for _ in range(n):
                    one_step()
            graphs[n] = g
        return graphs[n]

    def run_steps(k):
        if args.eager:
            for _ in range(k):
                one_step()
            return
        full, rest = divmod(k, per_graph)
        for _ in range(full):
            graph_of(per_graph).replay()
        if rest:
            graph_of(rest).replay()

    if not args.eager:
        graph_of(per_graph)
        if args.steps % per_graph:
            graph_of(args.steps % per_graph)
        run_steps(per_graph)
        barrier()
    t0, t1 = ev(), ev()
    with Clocks(local) as clk:
        run_steps(2 * per_graph)             # re-warm after the sampler's start-up idle gap
        barrier()
        t0.record(stream)
        run_steps(args.steps)
        t1.record(stream)
        barrier()
    ms_step = t0.elapsed_time(t1) / args.steps
    # sustained: >= 250 ms of back-to-back graph replays; HBM
    # streaming that long reaches the board power cap on this pool, so it is
    # reported beside the K-step headline with its own clock sample
    sustained = None
    if not (args.eager or args.profile):
        n_sus = max(per_graph, int(0.25 / max(ms_step * 1e-3, 1e-6)) // per_graph * per_graph)
        s0, s1 = ev(), ev()
        with Clocks(local) as clk_s:
            run_steps(2 * per_graph)
            barrier()
            s0.record(stream)
            run_steps(n_sus)
            s1.record(stream)
            barrier()
        ts = torch.tensor([s0.elapsed_time(s1) / n_sus], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        sustained = {"value": float(ts[0]) * 1e3, "unit": UNIT, "steps": n_sus,
                     "timed_ms": float(ts[0]) * n_sus, "clocks": clk_s.summary()}
    # per-replay distribution (graphs of `per_graph` steps, events between replays)
    rep_us = []
    if not args.eager:
        evs_r = [ev() for _ in range(min(args.steps // per_graph, 50) + 1)]
        barrier()
        evs_r[0].record(stream)
        for j in range(1, len(evs_r)):
            graph_of(per_graph).replay()
            evs_r[j].record(stream)
        barrier()
        rep_us = sorted(evs_r[j - 1].elapsed_time(evs_r[j]) * 1e3 / per_graph
                        for j in range(1, len(evs_r)))
    graphs.clear()
    # (2) the per-call breakdown (and the live roofline of score_select):
    #     another K steps with events between the calls
    n_brk = min(args.steps, 20)
    events = [[ev() for _ in range(4)] for _ in range(n_brk)]
    barrier()
    for i in range(n_brk):
        one_step(events[i])
    barrier()
    seg = [[e[j].elapsed_time(e[j + 1]) for e in events] for j in range(3)]
    per_step = sorted(e[0].elapsed_time(e[3]) * 1e3 for e in events)
    pct = lambda q: per_step[min(len(per_step) - 1, int(q * (len(per_step) - 1) + 0.5))]
    rq = lambda q: rep_us[min(len(rep_us) - 1, int(q * (len(rep_us) - 1) + 0.5))]
    avg_pred, avg_sel, avg_dec = (statistics.mean(s) for s in seg)
    t = torch.tensor([ms_step, avg_sel], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, avg_sel_max = float(t[0]), float(t[1])
    flags = int(step.dev_flags.item())

    # output all-gather (NCCL) timed separately: in a TP model o_proj consumes the shard
    gather_ms = None
    if world > 1:
        # head-major shards [Hq/P, B, Dv] -> the global [Hq, B, Dv] by one
        # all_gather_into_tensor (shard.gather_heads / gather_units)
        from paper_2510_07486_b200.shard import gather_units
        for _ in range(3):
            full = gather_units(step.out, sh, cfg.batch, cfg.n_q_heads, cfg.group)
        barrier()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(10):
            full = gather_units(step.out, sh, cfg.batch, cfg.n_q_heads, cfg.group)
        e1.record(stream)
        barrier()
        gather_ms = e0.elapsed_time(e1) / 10

    # e2e through the public API with host buffers (pinned): per step H2D of
    # the new query state q_t (fp32) and the new token's k/v rows; one a0
    # kernel (asyncspade_append) puts q_t into the window ring, bf16(q_t) into
    # the current query and the k/v rows into the caches; the step's decode
    # writes a double-buffered output that goes D2H.  The copies run on a
    # copy stream, overlapped with the previous step's compute (as a serving
    # loop would); every byte of every step still crosses PCIe inside the
    # timed region.
    e2e = None
    if not (args.no_e2e or args.profile):
        B, nq, D = sh.bn, step.n_q, cfg.head_dim
        L = cfg.seq_len
        h_qt = [torch.randn(B, nq, D, dtype=torch.float32).pin_memory() for _ in range(2)]
        h_kv = [torch.randn(2, B, step.n_kv, D).to(torch.bfloat16).pin_memory() for _ in range(2)]
        h_out = [torch.empty(B, nq, D, dtype=torch.float32).pin_memory() for _ in range(2)]
        d_qt = [torch.empty(B, nq, D, dtype=torch.float32, device="cuda") for _ in range(2)]
        d_kv = [torch.empty(2, B, step.n_kv, D, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
        d_out = [torch.empty(B, nq, D, dtype=torch.float32, device="cuda") for _ in range(2)]
        pos = step.seq_lens - 1                              # the newest slot of each row
        copy = torch.cuda.Stream()                            # H2D
        copy_out = torch.cuda.Stream()                        # D2H (both directions at once)
        h2d_done = [torch.cuda.Event() for _ in range(2)]
        used = [torch.cuda.Event() for _ in range(2)]
        out_ready = [torch.cuda.Event() for _ in range(2)]
        d2h_done = [torch.cuda.Event() for _ in range(2)]

        def h2d(i):
            b = i % 2
            with torch.cuda.stream(copy):
                copy.wait_event(used[b])                   # step i-2 consumed this buffer
                d_qt[b].copy_(h_qt[b], non_blocking=True)
                d_kv[b].copy_(h_kv[b], non_blocking=True)
                h2d_done[b].record(copy)

        def e2e_step(i):
            b = i % 2
            stream.wait_event(h2d_done[b])
            stream.wait_event(d2h_done[b])                   # step i-2's output left d_out[b]
            step.append(d_qt[b], d_kv[b][0], d_kv[b][1], pos)  # a0: one kernel
            used[b].record(stream)
            one_step(out=d_out[b])
            out_ready[b].record(stream)
            with torch.cuda.stream(copy_out):
                copy_out.wait_event(out_ready[b])
                h_out[b].copy_(d_out[b], non_blocking=True)
                d2h_done[b].record(copy_out)

        for i in range(2):
            used[i].record(stream)
            d2h_done[i].record(stream)
        h2d(0)
        for i in range(3):                                   # warm-up
            h2d(i + 1)
            e2e_step(i)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = ev(), ev()
        e0.record(stream)
        h2d(0)
        for i in range(args.steps):
            if i + 1 < args.steps:
                h2d(i + 1)
            e2e_step(i)
        stream.wait_stream(copy_out)                         # the last output is on the host
        e1.record(stream)
        barrier()
        tt = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        bi = h_qt[0].numel() * 4 + h_kv[0].numel() * 2
        bo = h_out[0].numel() * 4
        e2e = {"value": float(tt[0]) * 1e3, "unit": UNIT, "h2d_bytes_per_step": bi * world,
               "d2h_bytes_per_step": bo * world,
               "copies": "pinned host, one copy stream per direction, double-buffered, overlapped "
                         "with compute; "
                         "a0 (asyncspade_append) puts q_t / k / v into the state in one kernel"}

    # a5: the paper's steady state -- selection
    # for step t+1 (predict, score, top-k) on a side stream, overlapped with
    # step t's sparse attention on the main stream; the same four kernels per
    # step, reported beside the serial headline (no synthetic forward here).
    a5 = None
    if not (args.no_a5 or args.profile):
        from paper_2510_07486_b200.pipeline import AsyncPipeline
        del step
        torch.cuda.empty_cache()
        st1 = DecodeStep(cfg, "cuda", kv_heads=(h0, hn), n_fresh=1, window_dtype=wdt,
                         batch_range=(sh.b0, sh.bn))
        st1.fill_synthetic()
        st1.seq_lens.copy_(torch.tensor(lens, dtype=torch.int32))
        # the layer's other work: a weight-streaming synthetic forward of the
        # model's per-layer parameters (Qwen3-32B / Qwen3-8B, Table 1), 1/P per
        # GPU under P-way tensor parallelism
        lp = synth.QWEN3_32B_LAYER_PARAMS if cfg.n_q_heads == 64 else synth.QWEN3_8B_LAYER_PARAMS
        fwd_bytes = 0 if args.a5_no_forward else 2 * lp // shards
        pipe = AsyncPipeline(st1, forward_bytes=fwd_bytes, priority=args.a5_priority)
        res = {}
        for _ in range(3):
            pipe.forward(stream)
        barrier()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(args.steps):
            pipe.forward(stream)
        e1.record(stream)
        barrier()
        res["forward"] = e0.elapsed_time(e1) / args.steps * 1e3
        for name, fn in (("serial", pipe.run_step_serial), ("pipelined", pipe.run_step)):
            for _ in range(3):
                fn()
            pipe.drain()
            barrier()
            e0, e1 = ev(), ev()
            e0.record(stream)
            for _ in range(args.steps):
                fn()
            pipe.drain()
            e1.record(stream)
            barrier()
            tt = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            res[name] = float(tt[0]) * 1e3
        t_sel = (avg_pred + avg_sel) * 1e3
        a5 = {"serial_us": res["serial"], "pipelined_us": res["pipelined"],
              "forward_us": res["forward"], "forward_bytes": fwd_bytes, "unit": UNIT,
              "overlap_efficiency": ((res["serial"] - res["pipelined"]) / max(min(res["forward"], t_sel), 1e-9)
                                     if fwd_bytes else None),
              "pipelined_gain_frac": (res["serial"] - res["pipelined"]) / res["serial"],
              "what": "steady-state layer step: selection for t+1 (predict, score, top-k) on a "
                      "side stream overlapped with decode(t) and the layer's synthetic forward "
                      "(weight streaming, %.0f MB) on the main stream; serial = the same calls "
                      "on one stream; efficiency = (serial - pipelined) / min(forward, "
                      "selection)" % (fwd_bytes / 1e6)}
        del pipe, st1
        torch.cuda.empty_cache()

    if rank == 0:
        peak, peak_src = _peaks()
        D2 = cfg.head_dim * 2                          # per GPU: full-K + selected K and V
        k_bytes = sum(lens) * hn * D2
        # selected rows: K and V (absorbed MLA: one latent row serves both)
        n_sel_reads = 1 if cfg.v_head_dim and cfg.v_head_dim != cfg.head_dim else 2
        core = k_bytes + n_sel_reads * sum(min(cfg.top_k, n) for n in lens) * hn * D2
        achieved = k_bytes / (avg_sel_max * 1e-3) / 1e9
        # all algorithmic bytes: + the query window, q_hat written and
        # read, the current query, the indices written and read, the output
        n_q = sh.bn * hn * cfg.group
        wbytes = 2 if args.bf16_window else 4
        all_bytes = (core + n_q * cfg.window * cfg.head_dim * wbytes + 2 * n_q * cfg.head_dim * 4
                     + n_q * cfg.head_dim * 2 + 2 * sh.bn * hn * cfg.top_k * 4
                     + n_q * (cfg.v_head_dim or cfg.head_dim) * 4)
        line = {
            "metric": METRIC, "value": ms_step * 1e3, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16 KV, fp32 math (fp64 predictor)", "data": "synthetic",
            "config": {"workload": cfg.name, "batch": cfg.batch, "n_q_heads": cfg.n_q_heads,
                       "n_kv_heads": cfg.n_kv_heads, "head_dim": cfg.head_dim,
                       "seq_len": cfg.seq_len, "top_k": cfg.top_k, "window": cfg.window,
                       "query_window": "bf16" if args.bf16_window else "fp32",
                       "seq_lens": ("ragged: seeded uniform [L/8, L], mean %.0f" % (sum(lens) / len(lens))
                                    if args.ragged else "uniform L"),
                       "kv_layout": (f"paged: {args.paged}-token HND pages, random placement"
                                     if args.paged else "dense [B][Hkv][L][D]"),
                       "parallelism": (f"kv-head shard x{world}" if shards == world else
                                       f"emulated: rank 0 of a {shards}-way kv-head shard on 1 GPU")
                                      + ("" if sh.bn == cfg.batch else " (batch split)"),
                       "l2": "no flush: K+V per GPU (%.2f GB) >> 126 MB L2" %
                             (2 * k_bytes / 1e9)},
            "hbm_tb_per_s": core / (ms_step * 1e-3) / 1e12,
            "core_bytes_per_gpu": core,
            "all_bytes_per_gpu": all_bytes,
            "hbm_tb_per_s_all_bytes": all_bytes / (ms_step * 1e-3) / 1e12,
            "roofline_frac_step": core / (ms_step * 1e-3) / 1e9 / peak,
            "roofline_frac_step_nominal_8tbs": core / (ms_step * 1e-3) / 8e12,
            "per_call_ms": {"predict_query": avg_pred, "score_select": avg_sel,
                            "sparse_decode": avg_dec},
            "step_us_p10_p50_p90": ([rq(0.1), rq(0.5), rq(0.9)] if rep_us else
                                    [pct(0.1), pct(0.5), pct(0.9)]),
            "roofline": {"bound": "hbm", "kernel": "asyncspade_score_select (score + select)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic(),
                         "algorithmic_bytes_per_launch": k_bytes, "peak_source": peak_src},
            "gpu_launches": 5 * args.steps,
            "gpu_launches_e2e_per_step": 6,
            "timing": (("headline: CUDA-graph replays (%d steps per graph, PDL edges kept "
                        "inside), events around all K steps (%.0f ms timed); p10/p50/p90 of "
                        "per-replay times / %d; " % (per_graph, ms_step * args.steps, per_graph))
                       if not args.eager else "headline: events around K eager back-to-back "
                       "steps; ") + "per_call_ms / roofline: a second pass of %d eager steps "
                      "with events between the calls" % n_brk,
            "dev_flags": flags,
            "clocks": clk.summary(),
        }
        if sustained is not None:
            line["sustained"] = sustained
        if gather_ms is not None:
            line["allgather_out_ms"] = gather_ms
        if e2e is not None:
            line["e2e"] = e2e
        if a5 is not None:
            line["a5"] = a5
        if world == 1 and not (args.no_cpu_baseline or args.profile):
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

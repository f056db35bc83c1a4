"""Multi-process (gloo, world size 2) check of the KV-head-sharded path on CPU:
each rank builds ITS shard's inputs from the index-based generator, runs the
step (the CPU oracle stands in for the kernels here -- this test covers the
host-side sharding and the output gather, not the kernels), gathers the
outputs, and the result must equal the unsharded computation exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_07486_b200 import configs, shard, synth


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CFG = configs.QWEN3_8B.with_(batch=2, seq_len=512, top_k=64, window=8, head_dim=64)


# MQA (one KV head): two ranks split the batch
CFG_MQA = configs.Config("mqa-cpu", 0, 4, 8, 1, 64, 384, 48, 8)


def _shard_step(rank: int, world: int, cfg=CFG):
    """The rank's block of the step (head-major outputs [heads, batch, ...])."""
    import oracle
    seed = synth.base_seed(cfg.index)
    sh = shard.shard_units(cfg.batch, cfg.n_kv_heads, world, rank)
    q0, qn = sh.q_heads(cfg.group)
    win, q = synth.query_trace(seed, cfg.batch, cfg.n_q_heads, cfg.window, cfg.head_dim,
                               b0=sh.b0, batch_slice=sh.bn, h0=q0, head_slice=qn)
    K = synth.kv_cache(seed, synth.STREAM_K, cfg.batch, cfg.n_kv_heads, cfg.seq_len,
                       cfg.head_dim, b0=sh.b0, batch_slice=sh.bn, h0=sh.h0, head_slice=sh.hn)
    V = synth.kv_cache(seed, synth.STREAM_V, cfg.batch, cfg.n_kv_heads, cfg.seq_len,
                       cfg.head_dim, b0=sh.b0, batch_slice=sh.bn, h0=sh.h0, head_slice=sh.hn)
    _, _, idx, out = oracle.step(win, q, K, V, [cfg.seq_len] * sh.bn, cfg.top_k)
    return np.ascontiguousarray(idx.transpose(1, 0, 2)), np.ascontiguousarray(out.transpose(1, 0, 2)), sh


def _worker(rank, world, port, result_q, cfg=CFG):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx, out, sh = _shard_step(rank, world, cfg)
    full_out = shard.gather_units(torch.from_numpy(out), sh, cfg.batch, cfg.n_q_heads, cfg.group)
    full_idx = shard.gather_units(torch.from_numpy(idx), sh, cfg.batch, cfg.n_kv_heads, 1)
    if rank == 0:
        result_q.put((full_idx.numpy(), full_out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds():
    assert shard.shard_units(64, 8, 8, 3) == shard.Shard(0, 64, 3, 1)
    # P > Hkv: "by batch where heads run out" -- MQA over 8 ranks, 2 KV heads over 8
    assert [shard.shard_units(10, 1, 4, r) for r in range(4)] == [
        shard.Shard(0, 2, 0, 1), shard.Shard(2, 3, 0, 1), shard.Shard(5, 2, 0, 1), shard.Shard(7, 3, 0, 1)]
    assert shard.shard_units(64, 2, 8, 5) == shard.Shard(16, 16, 1, 1)
    with pytest.raises(ValueError):
        shard.shard_units(64, 8, 12, 0)
    assert shard.kv_head_shard(8, 1, 0) == (0, 8)
    assert [shard.kv_head_shard(8, 4, r) for r in range(4)] == [(0, 2), (2, 2), (4, 2), (6, 2)]
    assert shard.q_head_shard(64, 8, 8, 3) == (24, 8)
    with pytest.raises(ValueError):
        shard.kv_head_shard(8, 3, 0)


@pytest.mark.parametrize("cfg", [CFG, CFG_MQA], ids=["kv-head-split", "mqa-batch-split"])
def test_two_rank_gloo_sharded_step_matches_unsharded(cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, cfg)) for r in range(2)]
    for p in procs:
        p.start()
    idx, out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_idx, ref_out, _ = _shard_step(0, 1, cfg)
    np.testing.assert_array_equal(idx, ref_idx)
    np.testing.assert_array_equal(out, ref_out)


def _transport_worker(rank, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2510_07486_b200.disagg import Transport
    io = Transport(1 - rank)
    g = torch.Generator().manual_seed(3)
    pack = [torch.randn(2, 4, 8, generator=g), torch.randn(2, 2, 3, 8, generator=g).to(torch.bfloat16),
            torch.randint(-1, 100, (2, 3, 5), generator=g, dtype=torch.int32)]
    if rank == 0:                                    # Inference Rank: send the pack, get it back
        for t in pack:
            io.send(t)
        back = [torch.empty_like(t) for t in pack]
        for t in back:
            io.recv(t)
        result_q.put([bool(torch.equal(a.view(torch.uint8) if a.dtype == torch.bfloat16 else a,
                                       b.view(torch.uint8) if b.dtype == torch.bfloat16 else b))
                      for a, b in zip(pack, back)])
    else:                                            # Cache Rank: echo
        got = [torch.empty_like(t) for t in pack]
        for t in got:
            io.recv(t)
        for t in got:
            io.send(t)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_transport_is_bit_exact():
    """NEXT-1 host logic: the dual-rank Transport (gloo, raw-byte staging)
    moves fp32, bf16 and int32 packs bit for bit (a round trip)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transport_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok == [True, True, True]

"""KV-head sharding across GPUs.

Every unit of the hot path is independent end to end -- a1 per (b, q-head),
a2-a4 per (b, KV head) with its G q-heads -- so the step shards with no
exchange: rank r of P owns KV heads [r*Hkv/P, (r+1)*Hkv/P) and the matching q
heads for every batch row.  The only collective is the optional output
gather (a tensor-parallel model would feed its row-parallel o_proj directly).
"""
from __future__ import annotations


def kv_head_shard(n_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """(first KV head, number of KV heads) owned by `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if n_kv_heads % world:
        raise ValueError(f"{n_kv_heads} KV heads do not divide over {world} ranks")
    hn = n_kv_heads // world
    return rank * hn, hn


def q_head_shard(n_q_heads: int, n_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """(first q head, number of q heads) that go with the rank's KV heads."""
    h0, hn = kv_head_shard(n_kv_heads, world, rank)
    g = n_q_heads // n_kv_heads
    return h0 * g, hn * g


def gather_heads(shard, group=None):
    """All-gather per-rank [B, H_shard, ...] tensors into [B, H, ...] (rank-major
    head order == global head order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [torch.empty_like(shard) for _ in range(world)]
    dist.all_gather(parts, shard.contiguous(), group=group)
    return torch.cat(parts, dim=1)

"""Work partition across GPUs.

Every unit of the hot path is independent end to end -- a1 per (b, q-head),
a2-a4 per (b, KV head) with its G q-heads -- so the step shards with no
exchange.  Rank r of P owns:

* P <= Hkv (P divides Hkv): KV heads [r*Hkv/P, (r+1)*Hkv/P) and their q heads,
  for every batch row;
* P > Hkv (P a multiple of Hkv -- e.g. MQA / absorbed MLA with Hkv = 1,
  PAPER.md P:257): "by batch where heads run out" (BASELINE north star):
  the P ranks form Hkv groups of P/Hkv; group g owns KV head g and splits the
  batch into P/Hkv contiguous slices, rank r taking slice r % (P/Hkv).

The only collective is the optional output gather (a tensor-parallel model
would feed its row-parallel o_proj directly).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    b0: int          # first batch row
    bn: int          # batch rows
    h0: int          # first KV head
    hn: int          # KV heads

    def q_heads(self, group: int) -> tuple[int, int]:
        return self.h0 * group, self.hn * group


def shard_units(batch: int, n_kv_heads: int, world: int, rank: int) -> Shard:
    """The (batch, KV-head) block rank `rank` of `world` owns."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if world <= n_kv_heads:
        if n_kv_heads % world:
            raise ValueError(f"{n_kv_heads} KV heads do not divide over {world} ranks")
        hn = n_kv_heads // world
        return Shard(0, batch, rank * hn, hn)
    if world % n_kv_heads:
        raise ValueError(f"{world} ranks are not a multiple of {n_kv_heads} KV heads")
    per_head = world // n_kv_heads
    h, part = divmod(rank, per_head)
    b0 = batch * part // per_head
    b1 = batch * (part + 1) // per_head
    if b1 <= b0:
        raise ValueError(f"batch {batch} too small for {per_head} ranks per KV head")
    return Shard(b0, b1 - b0, h, 1)


def kv_head_shard(n_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """(first KV head, number of KV heads) owned by `rank` (P <= Hkv)."""
    s = shard_units(1, n_kv_heads, world, rank) if world <= n_kv_heads else None
    if s is None:
        raise ValueError(f"{n_kv_heads} KV heads do not divide over {world} ranks")
    return s.h0, s.hn


def q_head_shard(n_q_heads: int, n_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """(first q head, number of q heads) that go with the rank's KV heads."""
    h0, hn = kv_head_shard(n_kv_heads, world, rank)
    g = n_q_heads // n_kv_heads
    return h0 * g, hn * g


def gather_heads(shard, group=None):
    """All-gather per-rank HEAD-MAJOR outputs [H_shard, B, D] into [H, B, D].
    Rank r's heads follow rank r-1's, so the gather is one
    all_gather_into_tensor into a contiguous buffer -- a plain concatenation,
    no reordering (P <= Hkv)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    full = torch.empty((world * shard.shape[0],) + tuple(shard.shape[1:]), dtype=shard.dtype,
                       device=shard.device)
    dist.all_gather_into_tensor(full, shard.contiguous(), group=group)
    return full


def gather_units(shard_out, sh: Shard, batch: int, n_q_heads: int, group: int, pg=None):
    """All-gather per-rank head-major outputs [n_q(shard), b_n(shard), ...]
    into the full [n_q_heads, batch, ...].  P <= Hkv: a plain concatenation
    (gather_heads); P > Hkv (batch split): each rank's block is placed at its
    (q heads, batch slice)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(pg)
    if sh.bn == batch:
        return gather_heads(shard_out, pg)
    blocks = [torch.empty_like(shard_out) for _ in range(world)]   # equal slices required
    dist.all_gather(blocks, shard_out.contiguous(), group=pg)
    full = torch.empty((n_q_heads, batch) + tuple(shard_out.shape[2:]), dtype=shard_out.dtype,
                       device=shard_out.device)
    n_kv = n_q_heads // group
    for r, blk in enumerate(blocks):
        o = shard_units(batch, n_kv, world, r)
        q0, qn = o.q_heads(group)
        full[q0:q0 + qn, o.b0:o.b0 + o.bn] = blk
    return full

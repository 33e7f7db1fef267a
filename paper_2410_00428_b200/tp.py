"""KV-head sharding across GPUs.

Rank r of N owns KV heads [r*Hkv/N, (r+1)*Hkv/N) and their query heads
(GQA groups stay intact). The block table and free lists are replicated: every
rank runs the same KvManager call sequence, so slot ids agree. The only
exchange is an all-gather of per-head attention outputs after each layer.
"""
from __future__ import annotations


def kv_head_range(rank: int, world: int, n_kv_heads: int):
    if n_kv_heads % world:
        raise ValueError("world size must divide n_kv_heads")
    per = n_kv_heads // world
    return rank * per, (rank + 1) * per


def q_head_range(rank: int, world: int, n_heads: int, n_kv_heads: int):
    g = n_heads // n_kv_heads
    lo, hi = kv_head_range(rank, world, n_kv_heads)
    return lo * g, hi * g


def slot_bytes(tokens_per_block: int, kv_bytes_per_token_layer: int, world: int) -> int:
    """Bytes of one (block, layer) slot on one GPU: bs * kvB / TP."""
    return tokens_per_block * kv_bytes_per_token_layer // world


def assemble(gathered, world: int, batch: int, q_heads_local: int, head_dim: int):
    """[world * batch * hq_local * d] all-gather result -> [batch, world * hq_local, d]."""
    x = gathered.reshape(world, batch, q_heads_local, head_dim)
    return x.permute(1, 0, 2, 3).reshape(batch, world * q_heads_local, head_dim)


def all_gather_heads(dist, out_local, group=None):
    """The one collective of the path: all-gather per-head outputs
    [batch, hq_local, d] from every rank into [batch, hq, d]."""
    import torch
    world = dist.get_world_size(group)
    b, hql, d = out_local.shape
    buf = torch.empty((world * b * hql * d,), dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(buf, out_local.contiguous().reshape(-1), group=group)
    return assemble(buf, world, b, hql, d)

"""KV-head sharding of the hot path over N GPUs.

Rank i owns kv-heads [i*Hkv/N, (i+1)*Hkv/N) and their q-head groups; each rank runs its own
pool (same T-token logical chunking with T scaled by N so chunk_bytes stays a 2 MiB multiple;
allocation is deterministic, so every rank holds identical chunk tables). The only exchange is
the per-layer gather of the head-sharded attention outputs, over NCCL (torch.distributed).
"""
from __future__ import annotations


def head_partition(n_heads_q: int, n_heads_kv: int, world: int, rank: int):
    """(kv_begin, kv_end, q_begin, q_end) of `rank`. Requires world | n_heads_kv."""
    if world <= 0 or n_heads_kv % world or n_heads_q % n_heads_kv or not 0 <= rank < world:
        raise ValueError("KV heads must divide evenly over the ranks")
    hk = n_heads_kv // world
    group = n_heads_q // n_heads_kv
    return rank * hk, (rank + 1) * hk, rank * hk * group, (rank + 1) * hk * group


def shard_tokens_per_chunk(tokens_per_chunk_full: int, world: int) -> int:
    """T on each shard: chunk_bytes = 4*T*L*(Hkv/N)*d stays equal to the unsharded chunk."""
    return tokens_per_chunk_full * world


def gather_heads(out_local, world: int, group=None, out=None):
    """All-gather head-sharded attention outputs [B, Hq/N, d] -> [B, Hq, d] (rank-major heads,
    which is the global head order because ranks own contiguous head ranges)."""
    import torch
    import torch.distributed as dist
    B, hq, d = out_local.shape
    if world == 1:
        return out_local
    buf = torch.empty((world, B, hq, d), dtype=out_local.dtype, device=out_local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, out_local.contiguous(), group=group)
    else:
        dist.all_gather(list(buf.unbind(0)), out_local.contiguous(), group=group)
    full = buf.permute(1, 0, 2, 3).reshape(B, world * hq, d)
    if out is not None:
        out.copy_(full)
        return out
    return full

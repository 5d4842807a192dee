"""KV-head sharding of the hot path over N GPUs.

Rank i owns kv-heads [i*Hkv/N, (i+1)*Hkv/N) and their q-head groups; each rank runs its own
pool (same T-token logical chunking with T scaled by N so chunk_bytes stays a 2 MiB multiple;
allocation is deterministic, so every rank holds identical chunk tables). The only exchange is
the per-layer gather of the head-sharded attention outputs: fused into the attention
kernel's merge epilogue as peer-memory stores into every rank's window (PeerGather), with
`gather_heads` (NCCL all-gather) kept as the comparison path.
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


def gather_window_bytes(n_layers: int, batch: int, heads_q_total: int, head_dim: int) -> int:
    """Window size for one [B, Hq_total, d] bf16 output slot per layer (plus the flag words)."""
    from paper_2506_15155_b200.ellm import GATHER_DATA_OFFSET
    return GATHER_DATA_OFFSET + n_layers * layer_stride(batch, heads_q_total, head_dim)


def layer_stride(batch: int, heads_q_total: int, head_dim: int) -> int:
    """Bytes of one layer's gathered output [B, Hq_total, d] bf16 (16-B aligned)."""
    return (batch * heads_q_total * head_dim * 2 + 15) // 16 * 16


def exchange_handles(handle: bytes, world: int, group=None) -> list[bytes]:
    """All ranks' 64-byte IPC handles, rank order (torch.distributed object all-gather; works
    on gloo and nccl)."""
    import torch.distributed as dist
    if world == 1:
        return [bytes(handle)]
    out = [None] * world
    dist.all_gather_object(out, bytes(handle), group=group)
    return [bytes(h) for h in out]


class PeerGather:
    """a10 fused head gather over peer memory (include/ellm.h).

    Each rank allocates one gather window, the IPC handles are exchanged over the process
    group, every rank maps the others' windows (cudaIpcOpenMemHandle: NVLink P2P between the
    GPUs of one box) and attaches all N to its pool. From then on
    ``pool.attention_gather(l, ..., out_offset=self.offset(l))`` writes each finished output row
    straight into every rank's window and ``pool.gather_wait(l)`` orders the consumer after all
    ranks' rows — no separate collective launch. ``out(l)`` is the device address of layer l's
    gathered [B, Hq_total, d] rows in this rank's own window."""

    def __init__(self, pool, world: int, rank: int, heads_q_total: int, n_layers: int, batch: int,
                 head_dim: int, device: int, group=None):
        from paper_2506_15155_b200 import ellm
        self.ellm = ellm
        self.pool, self.world, self.rank = pool, world, rank
        self.stride = layer_stride(batch, heads_q_total, head_dim)
        self.nbytes = gather_window_bytes(n_layers, batch, heads_q_total, head_dim)
        self.own, handle = ellm.gather_window_create(device, self.nbytes)
        self.opened = []
        handles = exchange_handles(handle, world, group)
        windows = []
        for i, h in enumerate(handles):
            if i == rank:
                windows.append(self.own)
            else:
                a = ellm.ipc_open(h)
                self.opened.append(a)
                windows.append(a)
        self.windows = windows
        rc = pool.gather_attach(world, rank, heads_q_total, windows, self.nbytes)
        if rc != ellm.OK:
            self.close()
            raise ellm.EllmError(rc, "ellm_gather_attach")

    def offset(self, layer: int) -> int:
        return layer * self.stride

    def out(self, layer: int) -> int:
        return self.own + self.ellm.GATHER_DATA_OFFSET + self.offset(layer)

    def close(self):
        if self.pool is not None:
            self.pool.gather_detach()
        for a in self.opened:
            self.ellm.ipc_close(a)
        self.opened = []
        if self.own:
            self.ellm.gather_window_destroy(self.own)
            self.own = 0
        self.pool = None

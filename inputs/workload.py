"""Synthetic workloads of BASELINE.json (configs C1-C5) built through the product API.

Holds no method arithmetic: it sizes a pool for a config, draws K/V/Q with the seeded
counter-based generator (inputs/gen.cu on the device, bit-identical to inputs/gen.py), and
feeds them through libellm.so's own calls (kv_reserve / kv_append). Used by bench.py and by
the full-size parity tests; never imports the oracle.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
GEN_LIB = os.path.join(_HERE, "libellm_inputs.so")
_gen = None


def gen_lib():
    global _gen
    if _gen is None:
        if not os.path.exists(GEN_LIB):
            raise ImportError(f"{GEN_LIB} missing: run `python -m paper_2506_15155_b200.build`")
        _gen = ctypes.CDLL(GEN_LIB)
        V, I32, I64, U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        _gen.ellm_gen_kv.argtypes = [U64, I32, I64, I32, I32, I32, I32, I32, I32, I32, I64, V, V]
        _gen.ellm_gen_q.argtypes = [U64, I32, I32, I32, I32, I32, V, V]
    return _gen


@dataclasses.dataclass
class Workload:
    name: str
    n_layers: int
    n_heads_q: int
    n_heads_kv: int
    head_dim: int
    batch: int
    context: int
    seed: int
    tokens_per_chunk: int = 16
    world: int = 1
    rank: int = 0
    decode_headroom: int = 256   # extra tokens per request the pool can grow by
    needle: bool = True

    @property
    def group(self) -> int:
        return self.n_heads_q // self.n_heads_kv

    @property
    def hkv_local(self) -> int:
        return self.n_heads_kv // self.world

    @property
    def hq_local(self) -> int:
        return self.n_heads_q // self.world

    @property
    def kv_head0(self) -> int:
        return self.rank * self.hkv_local

    @property
    def q_head0(self) -> int:
        return self.rank * self.hq_local

    @property
    def needle_range(self) -> int:
        return self.context if self.needle else 0

    @property
    def chunks_per_request(self) -> int:
        T = self.tokens_per_chunk
        return (self.context + self.decode_headroom + T - 1) // T

    def chunk_bytes(self) -> int:
        return 4 * self.tokens_per_chunk * self.n_layers * self.hkv_local * self.head_dim

    def kv_bytes_per_layer(self, lens) -> int:
        """Algorithmic K+V bytes one attention launch reads."""
        return int(sum(lens)) * self.hkv_local * self.head_dim * 2 * 2


def c2(world=1, rank=0) -> Workload:
    """BASELINE.json configs[1]: LLaMA-3-8B shape, 32 requests x 32K, bf16 decode (seed 1).
    KV-head sharded: T*Hkv_local = 128 keeps 2 MiB chunks on every shard."""
    return Workload("c2-llama3-8b-32x32k", 32, 32, 8, 128, 32, 32768, seed=1,
                    tokens_per_chunk=16 * world, world=world, rank=rank)


def c4(world=1, rank=0, batch=64) -> Workload:
    """BASELINE.json configs[3]: LLaMA-70B shape, batch 64 x 8K (seed 3), T = 256/Hkv_local
    (10 MiB chunks on every shard)."""
    return Workload("c4-llama70b-64x8k", 80, 64, 8, 128, batch, 8192, seed=3,
                    tokens_per_chunk=32 * world, world=world, rank=rank)


def c3(batch=16) -> Workload:
    """BASELINE.json configs[2]: LLaMA-3-8B-262K shape, batch 16 x 128K context (seed 2): 256 GiB
    of KV in 2 MiB chunks, more than one B200 holds, so part of the batch lives in host slots."""
    return Workload("c3-llama3-8b-262k-16x128k", 32, 32, 8, 128, batch, 131072, seed=2,
                    tokens_per_chunk=16, decode_headroom=512)


def c5(batch=256) -> Workload:
    """BASELINE.json configs[4]: C5 churn at the LLaMA-3-8B shape: 256 requests, prompts 2K-128K
    (inputs/c5.py), 2 MiB chunks; the pool is smaller than the working set."""
    return Workload("c5-churn-8b-256req", 32, 32, 8, 128, batch, 131072, seed=5, tokens_per_chunk=16,
                    decode_headroom=256, needle=False)


def c1() -> Workload:
    return Workload("c1-tiny", 1, 4, 2, 64, 4, 300, seed=0, tokens_per_chunk=16, decode_headroom=64)


def make_pool(wl: Workload, device: int, host_slots: int = 0, extra_chunks: int = 0, extra_requests: int = 0):
    from paper_2506_15155_b200 import ellm
    nchunks = wl.batch * wl.chunks_per_request + extra_chunks
    return ellm.Pool(device, wl.n_layers, wl.hq_local, wl.hkv_local, wl.head_dim, wl.tokens_per_chunk,
                     nchunks, nchunks, wl.batch + extra_requests, wl.chunks_per_request, host_slots)


def fill_request(pool, wl: Workload, r: int, n: int, stream=None):
    """Reserve n tokens for request r and append all layers' K/V (device-generated)."""
    import torch
    from paper_2506_15155_b200 import ellm
    s = (stream or torch.cuda.current_stream()).cuda_stream
    rc = pool.reserve([r], [n], s)
    if rc != ellm.OK:
        raise ellm.EllmError(rc, "fill reserve")
    kb = torch.empty((n, wl.hkv_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    vb = torch.empty_like(kb)
    for layer in range(wl.n_layers):
        gen_kv_device(wl, r, 0, n, layer, 0, kb.data_ptr(), s)
        gen_kv_device(wl, r, 0, n, layer, 1, vb.data_ptr(), s)
        rc = pool.append(layer, [r], [n], kb, vb, s)
        if rc != ellm.OK:
            raise ellm.EllmError(rc, "fill append")
    torch.cuda.synchronize()


def gen_kv_device(wl: Workload, r: int, p0: int, n: int, layer: int, kv: int, out_ptr: int, stream=0):
    rc = gen_lib().ellm_gen_kv(wl.seed, r, p0, n, layer, kv, wl.kv_head0, wl.hkv_local, wl.head_dim,
                               wl.group, wl.needle_range, out_ptr, stream)
    if rc != 0:
        raise RuntimeError("ellm_gen_kv failed")


def gen_q_device(wl: Workload, r: int, layer: int, out_ptr: int, stream=0):
    rc = gen_lib().ellm_gen_q(wl.seed, r, layer, wl.q_head0, wl.hq_local, wl.head_dim, out_ptr, stream)
    if rc != 0:
        raise RuntimeError("ellm_gen_q failed")


def prefill(pool, wl: Workload, requests_per_batch: int | None = None, append_times: list | None = None):
    """Reserve `context` tokens for every request and append all layers' K/V through
    ellm_kv_append (bulk, prefill-sized appends), generated on the device. If `append_times`
    is a list, (seconds, bytes moved) of every append call is appended to it."""
    import torch
    from paper_2506_15155_b200 import ellm
    B, n, Hkv, d = wl.batch, wl.context, wl.hkv_local, wl.head_dim
    reqs = list(range(B))
    rc = pool.reserve(reqs, [n] * B)
    if rc != ellm.OK:
        raise ellm.EllmError(rc, "prefill reserve")
    rb = requests_per_batch or max(1, min(B, (1 << 30) // max(1, n * Hkv * d * 2)))
    kbuf = torch.empty((rb * n, Hkv, d), dtype=torch.bfloat16, device="cuda")
    vbuf = torch.empty_like(kbuf)
    row_bytes = Hkv * d * 2
    s = torch.cuda.current_stream().cuda_stream
    for layer in range(wl.n_layers):
        for r0 in range(0, B, rb):
            rs = reqs[r0:r0 + rb]
            for i, r in enumerate(rs):
                gen_kv_device(wl, r, 0, n, layer, 0, kbuf.data_ptr() + i * n * row_bytes, s)
                gen_kv_device(wl, r, 0, n, layer, 1, vbuf.data_ptr() + i * n * row_bytes, s)
            if append_times is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            rc = pool.append(layer, rs, [n] * len(rs), kbuf, vbuf, s)
            if rc != ellm.OK:
                raise ellm.EllmError(rc, f"prefill append layer {layer}")
            if append_times is not None:
                e1.record()
                append_times.append((e0, e1, 2 * 2 * len(rs) * n * Hkv * d * 2))  # K,V x read+write
    torch.cuda.synchronize()
    if append_times is not None:
        append_times[:] = [(a.elapsed_time(b) / 1e3, nb) for a, b, nb in append_times]


def decode_inputs(wl: Workload, step: int, lens):
    """Device tensors for one decode step: q [L, B, Hq_local, d], k/v [L, B, Hkv_local, d]
    (the new token of every request at position lens[r])."""
    import torch
    L, B = wl.n_layers, wl.batch
    q = torch.empty((L, B, wl.hq_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((L, B, wl.hkv_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    s = torch.cuda.current_stream().cuda_stream
    qrow = wl.hq_local * wl.head_dim * 2
    kvrow = wl.hkv_local * wl.head_dim * 2
    for layer in range(L):
        for r in range(B):
            gen_q_device(wl, r, layer, q[layer].data_ptr() + r * qrow, s)
            gen_kv_device(wl, r, int(lens[r]), 1, layer, 0, k[layer].data_ptr() + r * kvrow, s)
            gen_kv_device(wl, r, int(lens[r]), 1, layer, 1, v[layer].data_ptr() + r * kvrow, s)
    return q, k, v


def host_kv(wl: Workload, r: int, layer: int, length: int, via_device: bool | None = None):
    """numpy (K, V) [length, Hkv_local, d] bf16 bits of request r (the oracle side of the
    full-size parity checks). Drawn by inputs/gen.py, or — for long contexts, where numpy takes
    tens of seconds — by its bit-identical CUDA twin inputs/gen.cu (pinned against gen.py in
    tests/test_gpu_parity.py). Either way the values come from the input generator, never from
    the product path."""
    if via_device is None:
        via_device = length * wl.hkv_local * wl.head_dim > (1 << 24)
    if via_device:
        import torch
        out = []
        for kv in (0, 1):
            t = torch.empty((length, wl.hkv_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
            gen_kv_device(wl, r, 0, length, layer, kv, t.data_ptr(), torch.cuda.current_stream().cuda_stream)
            out.append(np_bits(t))
        return out[0], out[1]
    from inputs import gen
    heads = range(wl.kv_head0, wl.kv_head0 + wl.hkv_local)
    return gen.request_kv(wl.seed, r, length, layer, heads, wl.head_dim, wl.group, wl.needle_range)


def host_q(wl: Workload, r: int, layer: int):
    from inputs import gen
    return gen.q_bits(wl.seed, r, layer, range(wl.q_head0, wl.q_head0 + wl.hq_local), wl.head_dim)


def np_bits(t) -> np.ndarray:
    """bf16 torch tensor -> numpy uint16 bit patterns."""
    import torch
    return t.detach().view(torch.int16).cpu().numpy().view(np.uint16)

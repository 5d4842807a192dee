"""Time ellm_prefill_attention (f4) at 8B geometry: B requests whose last n_q positions attend
causally to a context of `ctx` tokens. Prints TFLOP/s (algorithmic causal flops) per config."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2506_15155_b200 import ellm  # noqa: E402


def run(B, ctx, n_q, Hq=32, Hkv=8, d=128, T=16, L=int(os.environ.get("PF_L", "1")), iters=10):
    chunks = B * ((ctx + T - 1) // T) + 8
    p = ellm.Pool(0, L, Hq, Hkv, d, T, chunks, chunks, B, (ctx + T - 1) // T + 1, 0)
    reqs = list(range(B))
    assert p.reserve(reqs, [ctx] * B) == 0
    k = torch.randn(B * ctx, Hkv, d, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(B * ctx, Hkv, d, device="cuda", dtype=torch.bfloat16)
    layer = L // 3  # a middle layer (its slab slot differs per chunk when slabs are rotated)
    assert p.append(layer, reqs, [ctx] * B, k, v) == 0  # only the layer read is filled
    q = torch.randn(B * n_q, Hq, d, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    scale = d ** -0.5
    for _ in range(2):
        assert p.prefill_attention(layer, reqs, [n_q] * B, q, out, scale) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        p.prefill_attention(layer, reqs, [n_q] * B, q, out, scale)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    keys = sum(ctx - n_q + i + 1 for i in range(n_q))  # per request per q-head
    flops = 4.0 * d * keys * Hq * B
    print(f"B={B} ctx={ctx} n_q={n_q}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s", flush=True)
    p.close()
    return flops / ms / 1e9


if __name__ == "__main__":
    for B, ctx, nq in [(1, 8192, 8192), (4, 4096, 4096), (8, 16384, 2048), (16, 2048, 2048), (2, 32768, 4096)]:
        run(B, ctx, nq)

"""Is C3's swap interference tied to the CUDA context that issues the host->device copy?
(DESIGN.md §5 C3, §10.) Times the C2-shape decode step (fused append + attention launches over
--batch x 32K requests; batch 32 = 128 GiB of KV read per step) alone and while ~1.5x its
duration of pinned host -> device copies (1 GiB each, into a separate 1 GiB device buffer) is
queued first on:
  same:     a second stream of the primary context (the pool's), via the driver API
  ctx2:     a stream of a second context on the same device (cuCtxCreate), via the driver API
The host buffer is cuMemHostAlloc(PORTABLE) so both contexts see it pinned. One JSON line per
variant: step ms and slowdown vs alone. (tools/interference.py: torch copies, same context;
tools/interference_ncu.sh: the copies in another process.)
  python tools/interference_ctx2.py [--batch 32]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402
from inputs import workload as W  # noqa: E402


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver error {err}")
    return r[1] if isinstance(r, tuple) and len(r) == 2 else (r[1:] if isinstance(r, tuple) else None)


ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--context", type=int, default=0)
ap.add_argument("--big-mapped-gib", type=int, default=0)
ap.add_argument("--kinds", default="")
a = ap.parse_args()
wl = W.c2()
wl.batch = a.batch
if a.context:
    wl.context = a.context
pool = W.make_pool(wl, 0)
W.prefill(pool, wl)
B, L = wl.batch, wl.n_layers
reqs, ones = list(range(B)), [1] * B
lens = np.full(B, wl.context, np.int64)
q, k, v = W.decode_inputs(wl, 0, lens)
out = torch.empty_like(q)
cs = torch.cuda.current_stream()
sp = cs.cuda_stream
scale = wl.head_dim ** -0.5

ck(cu.cuInit(0))
dev = ck(cu.cuDeviceGet(0))
prim = ck(cu.cuCtxGetCurrent())
N = 1 << 30
host = ck(cu.cuMemHostAlloc(N, cu.CU_MEMHOSTALLOC_PORTABLE))
# the pool's host slots are cudaHostAlloc(Mapped | Portable): a mapped copy of the same size, and
# optionally a large idle mapped region beside it (C3 pins 112 GiB of host slots)
host_m = ck(cu.cuMemHostAlloc(N, cu.CU_MEMHOSTALLOC_PORTABLE | cu.CU_MEMHOSTALLOC_DEVICEMAP))
big = ck(cu.cuMemHostAlloc(a.big_mapped_gib << 30, cu.CU_MEMHOSTALLOC_PORTABLE | cu.CU_MEMHOSTALLOC_DEVICEMAP)) \
    if a.big_mapped_gib else None
d_same = ck(cu.cuMemAlloc(N))
s_same = ck(cu.cuStreamCreate(cu.CUstream_flags.CU_STREAM_NON_BLOCKING))
ctx2 = ck(cu.cuCtxCreate(0, dev))  # becomes current
d_2 = ck(cu.cuMemAlloc(N))
s_2 = ck(cu.cuStreamCreate(cu.CUstream_flags.CU_STREAM_NON_BLOCKING))
ck(cu.cuCtxSetCurrent(prim))


def step():
    assert pool.reserve(reqs, ones, sp) == 0
    for l in range(L):
        assert pool.decode_append_attention(l, reqs, k[l], v[l], q[l], out[l], scale, sp) == 0


def side(kind, ms):
    n = max(1, int(ms / 19))  # ~19 ms per GiB at ~55 GB/s
    # (issuing context, destination buffer's context): same = (prim, prim), ctx2 = (ctx2, ctx2),
    # ctx2_to_prim = (ctx2, prim), prim_to_ctx2 = (prim, ctx2); ctx2_d2d: ctx2 H2D into its own
    # buffer, then a device -> device copy of it into the primary context's buffer (from ctx2)
    base = kind.replace("_mapped", "")
    # prim_to_ctx2_d2d: the primary context copies host -> the second context's buffer, then
    # device -> device into its own buffer (everything issued from the primary context)
    ctx, stream = (prim, s_same) if base in ("same", "prim_to_ctx2", "d2h", "prim_to_ctx2_d2d") else (ctx2, s_2)
    dst = d_same if base in ("same", "ctx2_to_prim") else d_2
    ck(cu.cuCtxSetCurrent(ctx))
    if kind == "ellm_upload":  # the library path: H2D into the side context's staging, then D2D
        for _ in range(n):
            assert pool.upload(int(d_same), int(host), N, stream=int(s_same)) == 0
        return
    hsrc = host_m if kind.endswith("_mapped") else host
    for _ in range(n):
        if kind.startswith("d2h"):  # device -> host from the primary context (a deflate's direction)
            ck(cu.cuMemcpyDtoHAsync(hsrc, d_same, N, stream))
            continue
        ck(cu.cuMemcpyHtoDAsync(dst, hsrc, N, stream))
        if base in ("ctx2_d2d", "prim_to_ctx2_d2d"):
            ck(cu.cuMemcpyDtoDAsync(d_same, d_2, N, stream))
    ck(cu.cuCtxSetCurrent(prim))


def timed(kind):
    torch.cuda.synchronize()
    ck(cu.cuCtxSetCurrent(ctx2))
    ck(cu.cuCtxSynchronize())
    ck(cu.cuCtxSetCurrent(prim))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if kind:
        side(kind, 20.0 * a.steps * 1.5)
    e0.record(cs)
    for _ in range(a.steps):
        step()
    e1.record(cs)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / a.steps
    ck(cu.cuCtxSetCurrent(ctx2))
    ck(cu.cuCtxSynchronize())
    ck(cu.cuCtxSetCurrent(prim))
    torch.cuda.synchronize()
    return t


step()
base = timed(None)
for rep in range(2):
    kinds = [None] + [k for k in a.kinds.split(",") if k] if a.kinds else \
        ([None, "same", "ctx2", "ctx2_to_prim", "prim_to_ctx2", "ctx2_d2d", "d2h"] if rep == 0 else [None, "ctx2_d2d", "d2h"])
    for kind in kinds:
        t = timed(kind)
        print(json.dumps({"variant": kind or "alone", "batch": B, "kv_gib": B * wl.context * 128 * 1024 / 2 ** 30,
                          "step_ms": round(t, 3), "slowdown": round(t / base, 3)}), flush=True)

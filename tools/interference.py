"""What slows the decode attention when a host->device copy runs beside it (C3's swap
interference)? Times one C2 decode step (32 fused append + attention launches over
`--batch` x 32K requests) alone and with a concurrent side-stream writer of about the host link's
rate: (h2d) pinned host -> device copies, (d2h) device -> host copies, (wr) device-side writes of
4 MiB fills paced by spin kernels to a similar byte rate, (wr_fast) unpaced device fills.
Prints one JSON line per variant: step ms and slowdown vs alone.

  python tools/interference.py [--batch 32]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from inputs import workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--pad-gib", type=int, default=0, help="extra idle device allocation (GiB)")
ap.add_argument("--only", default="", help="comma-separated variants (default: all)")
a = ap.parse_args()
wl = W.c2()
wl.batch = a.batch
pad = torch.empty(a.pad_gib << 30, dtype=torch.uint8, device="cuda") if a.pad_gib else None
pool = W.make_pool(wl, 0)
W.prefill(pool, wl)
B, L = wl.batch, wl.n_layers
reqs, ones = list(range(B)), [1] * B
lens = np.full(B, wl.context, np.int64)
q, k, v = W.decode_inputs(wl, 0, lens)
out = torch.empty_like(q)
cs = torch.cuda.current_stream()
sp = cs.cuda_stream
side = torch.cuda.Stream()
scale = wl.head_dim ** -0.5


def step():
    assert pool.reserve(reqs, ones, sp) == 0
    for l in range(L):
        assert pool.decode_append_attention(l, reqs, k[l], v[l], q[l], out[l], scale, sp) == 0


N = 1 << 30
hbuf = torch.empty(N, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(N, dtype=torch.uint8, device="cuda")
fill = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")


def side_work(kind, ms):
    """Enqueue ~ms of side-stream traffic."""
    with torch.cuda.stream(side):
        if kind == "h2d":
            for _ in range(max(1, int(ms / 19))):  # ~19 ms per GiB at ~55 GB/s
                dbuf.copy_(hbuf, non_blocking=True)
        elif kind == "d2h":
            for _ in range(max(1, int(ms / 18))):
                hbuf.copy_(dbuf, non_blocking=True)
        elif kind == "wr":  # 4 MiB fill then ~70 us spin: ~55 GB/s of HBM writes
            for _ in range(int(ms / 0.075)):
                fill.fill_(1)
                torch.cuda._sleep(100000)
        elif kind == "wr_fast":
            for _ in range(int(ms * 1000)):
                fill.fill_(1)


def timed(kind):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if kind:
        side_work(kind, 20.0 * a.steps * 1.5)
    e0.record(cs)
    for _ in range(a.steps):
        step()
    e1.record(cs)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps


step()
base = timed(None)
kinds = [None] + ([k for k in a.only.split(",") if k] or ["h2d", "d2h", "wr", "wr_fast"])
for kind in kinds:
    t = timed(kind)
    print(json.dumps({"variant": kind or "alone", "batch": B, "kv_gib": round(B * wl.context * 128 * 1024 / 2 ** 30, 1),
                      "pad_gib": a.pad_gib, "step_ms": round(t, 3), "slowdown": round(t / base, 3)}), flush=True)

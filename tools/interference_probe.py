"""Decode-attention launches of the C2 shape at --batch x 32K (batch 32 = 128 GiB of KV read per
step, 24 = 96 GiB) for the two-process interference probe (tools/interference_ncu.sh). Times
--steps decode steps with CUDA events (printed as one JSON line), then, inside a
cudaProfilerStart/Stop range, runs --profiled more fused append + attention launches for ncu."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from inputs import workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--profiled", type=int, default=0)
ap.add_argument("--label", default="")
a = ap.parse_args()
wl = W.c2()
wl.batch = a.batch
pool = W.make_pool(wl, 0)
W.prefill(pool, wl)
B, L = wl.batch, wl.n_layers
reqs, ones = list(range(B)), [1] * B
lens = np.full(B, wl.context, np.int64)
q, k, v = W.decode_inputs(wl, 0, lens)
out = torch.empty_like(q)
sp = torch.cuda.current_stream().cuda_stream
scale = wl.head_dim ** -0.5


def step(layers=L):
    assert pool.reserve(reqs, ones, sp) == 0
    for l in range(layers):
        assert pool.decode_append_attention(l, reqs, k[l], v[l], q[l], out[l], scale, sp) == 0


step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
print(json.dumps({"label": a.label, "batch": B, "kv_gib": B * wl.context * 128 * 1024 / 2 ** 30,
                  "step_ms": round(ms, 3), "launch_us": round(ms / L * 1e3, 1)}), flush=True)
if a.profiled:
    torch.cuda.cudart().cudaProfilerStart()
    step(a.profiled)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()

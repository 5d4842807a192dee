"""Where does the pipelined end-to-end decode step lose time? C2 shape, fused PDL decode step with
each step's Q / new K,V uploaded from pinned host memory and its output read back, variants:
  serial        torch copies on the compute stream (bench.py's round-2 e2e)
  pipe          uploads via ellm_upload on a second stream one step ahead, read-back on a third
  pipe_torchup  as pipe, uploads with torch copies (host-link writes into the decode context)
  pipe_nodl     as pipe, read-back on the compute stream
  noio          the same loop with no host copies (device-resident inputs)
python tools/e2e_probe.py [steps] [c2|c4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from inputs import workload as W  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
wl = W.c4() if len(sys.argv) > 2 and sys.argv[2] == "c4" else W.c2()
pool = W.make_pool(wl, 0)
pool.set_launch_overlap(True)
W.prefill(pool, wl)
B, L = wl.batch, wl.n_layers
reqs, ones = list(range(B)), [1] * B
lens = np.full(B, wl.context, np.int64)
scale = wl.head_dim ** -0.5
cs = torch.cuda.current_stream()
sp = cs.cuda_stream
dev0 = W.decode_inputs(wl, 0, lens)
hin = [tuple(x.cpu().pin_memory() for x in W.decode_inputs(wl, j, lens + j)) for j in range(2)]
dev_in = [tuple(torch.empty_like(x) for x in dev0) for _ in range(2)]
outs = [torch.empty_like(dev0[0]) for _ in range(2)]
hout = [torch.empty(outs[0].shape, dtype=outs[0].dtype).pin_memory() for _ in range(2)]
up, dn = torch.cuda.Stream(), torch.cuda.Stream()
assert pool.upload(dev_in[0][0], hin[0][0]) == 0  # side context created outside the timed runs


def step(q, k, v, o):
    assert pool.reserve(reqs, ones, sp) == 0
    for l in range(L):
        assert pool.decode_append_attention(l, reqs, k[l], v[l], q[l], o[l], scale, sp) == 0


def run(mode):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    ev_up, ev_used, ev_dl = [None, None], [None, None], [None, None]

    def upload(j):
        b = j % 2
        if ev_used[b] is not None:
            up.wait_event(ev_used[b])
        for dt, ht in zip(dev_in[b], hin[j % 2]):
            if mode == "pipe_torchup":
                with torch.cuda.stream(up):
                    dt.copy_(ht, non_blocking=True)
            else:
                assert pool.upload(dt, ht, stream=up.cuda_stream) == 0
        ev_up[b] = torch.cuda.Event()
        ev_up[b].record(up)

    if mode.startswith("pipe"):
        up.wait_event(e0)
        upload(0)
    for j in range(steps):
        b = j % 2
        if mode == "noio":
            step(*dev_in[b], outs[b])
            continue
        if mode == "serial":
            for dt, ht in zip(dev_in[b], hin[b]):
                dt.copy_(ht, non_blocking=True)
            step(*dev_in[b], outs[b])
            hout[b].copy_(outs[b], non_blocking=True)
            continue
        cs.wait_event(ev_up[b])
        if ev_dl[b] is not None:
            cs.wait_event(ev_dl[b])
        step(*dev_in[b], outs[b])
        ev_used[b] = torch.cuda.Event()
        ev_used[b].record(cs)
        if j + 1 < steps:
            upload(j + 1)
        if mode == "pipe_nodl":
            hout[b].copy_(outs[b], non_blocking=True)
        else:
            dn.wait_event(ev_used[b])
            with torch.cuda.stream(dn):
                hout[b].copy_(outs[b], non_blocking=True)
            ev_dl[b] = torch.cuda.Event()
            ev_dl[b].record(dn)
    cs.wait_stream(dn)
    cs.wait_stream(up)
    e1.record(cs)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


run("noio")
for rep in range(2):
    for mode in ["noio", "serial", "pipe", "pipe_torchup", "pipe_nodl"]:
        print(f"{mode:13s} {run(mode):7.3f} ms/step", flush=True)

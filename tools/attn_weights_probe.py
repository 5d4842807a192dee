"""Can a static per-CTA weighting remove the streaming-time spread of the decode attention?
(PDL off, so each CTA stays on its SM from launch to launch.) Phase 0: equal shares, traced;
then weights = measured per-CTA rates, traced; then one multiplicative refinement, traced.
python tools/attn_weights_probe.py [c2|c4] [shard N]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15155_b200 import ellm  # noqa: E402
from inputs import workload as W  # noqa: E402


def main():
    wname = sys.argv[1] if len(sys.argv) > 1 else "c4"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    pdl = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    wl = W.c4(n, 0) if wname == "c4" else W.c2(n, 0)
    pool = W.make_pool(wl, 0)
    pool.set_launch_overlap(bool(pdl))
    W.prefill(pool, wl)
    L, B = wl.n_layers, wl.batch
    reqs, ones = list(range(B)), [1] * B
    out = torch.empty((L, B, wl.hq_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    G = torch.cuda.get_device_properties(0).multi_processor_count
    sp = torch.cuda.current_stream().cuda_stream
    scale = 1.0 / np.sqrt(wl.head_dim)
    state = {"s": 0}
    lens0 = np.full(B, wl.context, np.int64)

    def run(steps, trace):
        buf = torch.zeros((steps * L, G, 8), dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        if trace:
            assert pool.set_attn_trace(buf, steps * L) == 0
        for _ in range(steps):
            s = state["s"]
            q, k, v = W.decode_inputs(wl, s % 4, lens0 + s)
            assert pool.reserve(reqs, ones, sp) == 0
            for l in range(L):
                assert pool.decode_append_attention(l, reqs, k[l], v[l], q[l], out[l], scale, sp) == 0
            state["s"] += 1
        torch.cuda.synchronize()
        pool.set_attn_trace(None, 0)
        return buf.cpu().numpy()

    def summary(t, label):
        spans, ends, durs = [], [], []
        per = [(t[i + 1][:, 0].min() - t[i][:, 0].min()) / 1e3 for i in range(t.shape[0] - 1)]
        for i in range(t.shape[0]):
            x = t[i]
            t0 = x[:, 0].min()
            spans.append((x[:, 5].max() - t0) / 1e3)
            e = (x[:, 3] - t0) / 1e3
            ends.append((e.min(), np.median(e), e.max()))
            durs.append(x[:, 3] - x[:, 2])
        e = np.median(np.array(ends), axis=0)
        d = np.median(np.array(durs), axis=0)
        print(f"{label:28s} period {np.median(per):8.2f} span {np.median(spans):8.2f} us; streaming end min/med/max {e[0]:.2f} / {e[1]:.2f} / "
              f"{e[2]:.2f} us; per-CTA duration / median: {d.min() / np.median(d):.3f} .. {d.max() / np.median(d):.3f}")
        return d

    run(2, False)
    d0 = summary(run(2, True), f"{wl.name} x{n} pdl {pdl} equal shares")
    w = np.full(G, 1.0)
    share = np.full(G, 1.0)
    d = d0
    for it in range(3):
        rate = share / d            # tiles (relative) per ns
        w = rate / rate.mean()
        assert pool.debug_attn_weights(w) == 0
        run(1, False)
        share = w
        d = summary(run(2, True), f"weights, iteration {it + 1}")
    assert pool.debug_attn_weights([]) == 0
    summary(run(2, True), "equal shares again")
    pool.close()


if __name__ == "__main__":
    main()

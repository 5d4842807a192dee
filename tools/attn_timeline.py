"""Per-CTA timeline of back-to-back attention launches (ellm_set_attn_trace): where the time of a
small (sharded) decode launch goes. python tools/attn_timeline.py [c2|c4] [shard N] [p2p|none] [pdl 0|1]

Prints, per launch (medians over the traced steps, microseconds, relative to the launch's first
CTA start): the span (first start -> last end), the spread of CTA starts, the producer's PDL wait,
the first data, the streaming end (min / median / max over CTAs), merges, the last end, and the
gap to the next launch's first start (negative = overlap)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15155_b200 import ellm, shard  # noqa: E402
from inputs import workload as W  # noqa: E402


def main():
    wname = sys.argv[1] if len(sys.argv) > 1 else "c4"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    mode = sys.argv[3] if len(sys.argv) > 3 else "p2p"
    pdl = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    wl = W.c4(n, 0) if wname == "c4" else W.c2(n, 0)
    pool = W.make_pool(wl, 0)
    pool.set_launch_overlap(bool(pdl))
    W.prefill(pool, wl)
    L, B = wl.n_layers, wl.batch
    reqs, ones = list(range(B)), [1] * B
    lens = np.full(B, wl.context, np.int64)
    steps, warm = 2, 4
    ins = [W.decode_inputs(wl, s, lens + s) for s in range(warm + steps)]
    out = torch.empty((L, B, wl.hq_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    pg = shard.PeerGather(pool, 1, 0, wl.hq_local, L, B, wl.head_dim, device=0) if mode == "p2p" else None
    G = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros((steps * L, G, 8), dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    scale = 1.0 / np.sqrt(wl.head_dim)
    for s in range(warm + steps):
        if s == warm:
            torch.cuda.synchronize()
            assert pool.set_attn_trace(buf, steps * L) == 0
        q, k, v = ins[s]
        assert pool.reserve(reqs, ones, sp) == 0
        for l in range(L):
            if pg is not None:
                if l > 0:
                    assert pool.gather_wait_next(l - 1) == 0
                assert pool.attention_gather(l, reqs, q[l], pg.offset(l), scale, k[l], v[l], sp) == 0
            else:
                assert pool.decode_append_attention(l, reqs, k[l], v[l], q[l], out[l], scale, sp) == 0
        if pg is not None:
            assert pool.gather_wait(L - 1, sp) == 0
    torch.cuda.synchronize()
    pool.set_attn_trace(None, 0)
    t = buf.cpu().numpy().astype(np.int64)
    G_used = int((t[0, :, 0] > 0).sum())
    t = t[:, :G_used]
    rows = []
    for i in range(t.shape[0]):
        x = t[i]
        t0 = x[:, 0].min()
        rel = lambda c: (x[:, c] - t0) / 1e3  # noqa: E731
        merged = x[:, 6] > 0
        r = {"span": (x[:, 5].max() - t0) / 1e3, "start_spread": rel(0).max(), "pdl_wait": np.median(rel(1)),
             "first_data": np.median(rel(2)), "stream_end_min": rel(3).min(), "stream_end_med": np.median(rel(3)),
             "stream_end_max": rel(3).max(), "merge_us": np.median((x[merged, 4] - x[merged, 3]) / 1e3) if merged.any() else 0,
             "end_max": rel(5).max(), "end_med": np.median(rel(5))}
        if i + 1 < t.shape[0]:
            r["gap_next"] = (t[i + 1][:, 0].min() - x[:, 5].max()) / 1e3
        rows.append(r)
    keys = list(rows[0])
    print(f"{wl.name} shard x{n} ({G_used} CTAs), gather {mode}, pdl {pdl}: medians over {len(rows)} launches (us)")
    for k in keys:
        vals = [r[k] for r in rows if k in r]
        print(f"  {k:16s} {statistics.median(vals):8.2f}   (min {min(vals):7.2f}, max {max(vals):7.2f})")
    # is a CTA's streaming time a property of its SM? per SM id: mean over launches of
    # (streaming end - first data) relative to the launch median; correlation of two halves
    dur = {}
    for i in range(t.shape[0]):
        x = t[i]
        d = (x[:, 3] - x[:, 2]).astype(np.float64)
        d /= np.median(d)
        for c in range(x.shape[0]):
            dur.setdefault(int(x[c, 7]), []).append(d[c])
    sms = sorted(dur)
    a = np.array([np.mean(dur[s][0::2]) for s in sms])
    b = np.array([np.mean(dur[s][1::2]) for s in sms])
    print(f"  per-SM streaming time / launch median: min {a.min():.3f} max {a.max():.3f}; "
          f"even/odd-launch correlation {np.corrcoef(a, b)[0, 1]:.3f}")
    same = np.mean([np.mean(t[i][:, 7] == t[0][:, 7]) for i in range(t.shape[0])])
    print(f"  CTA -> SM mapping equal to the first traced launch's: {same:.3f} of CTAs on average")
    bdur = np.array([(t[i][:, 3] - t[i][:, 2]) / np.median(t[i][:, 3] - t[i][:, 2]) for i in range(t.shape[0])])
    ba, bb = bdur[0::2].mean(0), bdur[1::2].mean(0)
    print(f"  per-CTA (blockIdx) streaming time ratio: min {ba.min():.3f} max {ba.max():.3f}; "
          f"even/odd correlation {np.corrcoef(ba, bb)[0, 1]:.3f}")
    slow = sorted(zip(((a + b) / 2).round(3), sms))[-6:]
    print("  slowest SMs (ratio, smid):", slow)
    if pg is not None:
        pg.close()
    pool.close()


if __name__ == "__main__":
    main()

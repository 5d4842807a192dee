"""With PDL the CTAs of launch k+1 start on SMs in the order launch k's CTAs exit, so high block
indices start last. Does giving them less static work (weights 1 - a*b/(G-1)) shorten the period?
python tools/ramp_probe.py [c2|c4] [shard N]  (PDL on, device-timed per-launch period)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import workload as W  # noqa: E402


def main():
    wname = sys.argv[1] if len(sys.argv) > 1 else "c4"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    wl = W.c4(n, 0) if wname == "c4" else W.c2(n, 0)
    pool = W.make_pool(wl, 0)
    pool.set_launch_overlap(True)
    W.prefill(pool, wl)
    L, B = wl.n_layers, wl.batch
    reqs, ones = list(range(B)), [1] * B
    out = torch.empty((L, B, wl.hq_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    G = torch.cuda.get_device_properties(0).multi_processor_count
    sp = torch.cuda.current_stream().cuda_stream
    scale = 1.0 / np.sqrt(wl.head_dim)
    lens0 = np.full(B, wl.context, np.int64)
    ins = [W.decode_inputs(wl, s, lens0 + s) for s in range(4)]
    state = {"s": 0}

    def steps(k):
        for _ in range(k):
            s = state["s"]
            q, kk, v = ins[s % 4]
            assert pool.reserve(reqs, ones, sp) == 0
            for l in range(L):
                assert pool.decode_append_attention(l, reqs, kk[l], v[l], q[l], out[l], scale, sp) == 0
            state["s"] += 1

    for a in [0.0, 0.03, 0.06, 0.1, 0.15, 0.0]:
        w = 1.0 - a * np.arange(G) / (G - 1)
        assert pool.debug_attn_weights(w if a > 0 else []) == 0
        steps(2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        steps(6)
        e1.record()
        torch.cuda.synchronize()
        print(f"{wl.name} x{n} ramp a={a:.2f}: {e0.elapsed_time(e1) * 1e3 / (6 * L):.2f} us per launch", flush=True)
    pool.close()


if __name__ == "__main__":
    main()

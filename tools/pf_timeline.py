"""Hand-off timeline of the f4 prefill kernel (first CTA, key tiles 0..15, clock64 cycles):
softmax of Q tile x waits S_x(t) -> works -> arrives P_x(t); the MMA thread sees P_x(t) -> issues
P_x.V and S_x(t+1). Prints medians over tiles 3..13. python tools/pf_timeline.py [lib variant env]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15155_b200 import ellm  # noqa: E402


def main():
    B, ctx, n_q, Hq, Hkv, d, T = 2, 32768, 4096, 32, 8, 128, 16
    chunks = B * ((ctx + T - 1) // T) + 8
    p = ellm.Pool(0, 1, Hq, Hkv, d, T, chunks, chunks, B, (ctx + T - 1) // T + 1, 0)
    reqs = list(range(B))
    assert p.reserve(reqs, [ctx] * B) == 0
    k = torch.randn(B * ctx, Hkv, d, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(B * ctx, Hkv, d, device="cuda", dtype=torch.bfloat16)
    assert p.append(0, reqs, [ctx] * B, k, v) == 0
    q = torch.randn(B * n_q, Hq, d, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    assert p.prefill_attention(0, reqs, [n_q] * B, q, out, d ** -0.5) == 0
    G = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros((1, G, 8), dtype=torch.int64, device="cuda")
    assert p.set_attn_trace(buf, 1) == 0
    assert p.prefill_attention(0, reqs, [n_q] * B, q, out, d ** -0.5) == 0
    torch.cuda.synchronize()
    p.set_attn_trace(None, 0)
    t = buf.view(-1)[: 16 * 16].cpu().numpy().reshape(16, 16).astype(np.int64)
    rng = range(3, 14)
    med = lambda a: float(np.median(a))  # noqa: E731
    print("per key tile (cycles, medians over tiles 3..13):")
    print(f"  softmax Q0: S ready -> P stored        {med([t[i, 1] - t[i, 0] for i in rng]):8.0f}")
    print(f"  softmax Q1: S ready -> P stored        {med([t[i, 3] - t[i, 2] for i in rng]):8.0f}")
    print(f"  P0 stored -> MMA thread sees it        {med([t[i, 4] - t[i, 1] for i in rng]):8.0f}")
    print(f"  P1 stored -> MMA thread sees it        {med([t[i, 6] - t[i, 3] for i in rng]):8.0f}")
    print(f"  MMA: P0.V + S0(t+1) issued (issue time)  {med([t[i, 5] - t[i, 4] for i in rng]):8.0f}")
    print(f"  S0(t+1) issued -> softmax Q0 sees S    {med([t[i + 1, 0] - t[i, 5] for i in rng]):8.0f}")
    print(f"  S1(t+1) issued -> softmax Q1 sees S    {med([t[i + 1, 2] - t[i, 7] for i in rng]):8.0f}")
    print(f"  period (softmax Q0 S-ready to S-ready) {med([t[i + 1, 0] - t[i, 0] for i in rng]):8.0f}")
    print(f"  Q1 S-ready minus Q0 S-ready (phase)    {med([t[i, 2] - t[i, 0] for i in rng]):8.0f}")
    if t[:, 8].any() and not t[:, 11].any():  # softmax-phase stamps (Q0, first warp)
        print(f"  softmax Q0: S ready -> S in registers  {med([t[i, 8] - t[i, 0] for i in rng]):8.0f}")
        print(f"  softmax Q0: -> pair max exchanged      {med([t[i, 9] - t[i, 8] for i in rng]):8.0f}")
        print(f"  softmax Q0: -> P stored (exps, st)     {med([t[i, 10] - t[i, 9] for i in rng]):8.0f}")
    if not t[:, 11:].any():  # the MMA-loop / producer stamps exist only in some kernel versions
        p.close()
        return
    print(f"  MMA loop: top -> V(t) ready            {med([t[i, 9] - t[i, 8] for i in rng]):8.0f}")
    print(f"  MMA loop: V(t) -> K(t+2) ready         {med([t[i, 10] - t[i, 9] for i in rng]):8.0f}")
    print(f"  MMA loop: K ready -> P0 seen           {med([t[i, 4] - t[i, 10] for i in rng]):8.0f}")
    print(f"  MMA loop: S1 issued -> next top        {med([t[i + 1, 8] - t[i, 7] for i in rng]):8.0f}")
    print(f"  producer: issue K(t+2)                 {med([t[i, 12] - t[i, 11] for i in rng]):8.0f}")
    print(f"  producer: issue V(t)                   {med([t[i, 13] - t[i, 12] for i in rng]):8.0f}")
    print(f"  producer iteration                     {med([t[i + 1, 11] - t[i, 11] for i in rng]):8.0f}")
    print(f"  V(t) issued by producer -> MMA sees V  {med([t[i, 9] - t[i, 13] for i in rng]):8.0f}")
    print(f"  issue V(t): start -> empty slot seen   {med([t[i, 14] - t[i, 12] for i in rng]):8.0f}")
    print(f"  issue V(t): empty seen -> TMAs issued  {med([t[i, 15] - t[i, 14] for i in rng]):8.0f}")
    p.close()


if __name__ == "__main__":
    main()

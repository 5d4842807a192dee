"""Small end-to-end cases of every kernel family, for compute-sanitizer:

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tests/sanitize_cases.py CASE

CASE: c1 (C1 flow: reserve / append / deflate / inflate through both swap engines / migrate
through the TMA bulk kernel / attention), pdl (fused decode launches back to back with
programmatic dependent launch on a full grid), gather (N = 2 shard pools in one process, fused
head gather with folded waits), prefill (f4 tcgen05 chunked prefill). Every case also checks
its results against the oracle (tests/twin.py), so a clean sanitizer log is a log of a correct
run. Test infrastructure: run by tools/sanitize.sh, not by pytest."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def case_c1():
    from tests.twin import Twin
    t = Twin(1, 4, 2, 64, 16, 64, 64, 4, 32, 16, seed=0)
    lens = [17, 64, 129, 300]
    assert t.reserve([0, 1, 2, 3], lens) == 0
    t.append_all_layers([0, 1, 2, 3], lens)
    for mode in (0, 1, 2, 3):
        assert t.p.set_swap_mode(mode) == 0
        rc, slots = t.deflate(t.o.table(3)[0][:8].tolist())
        assert rc == 0
        assert t.inflate(slots)[0] == 0
    t.check_tables()
    t.check_bytes()
    t.attention(0, [0, 1, 2, 3])
    # 8B-shaped pool with 32 KiB chunks: migrate goes through the TMA bulk copy kernel
    t2 = Twin(2, 32, 8, 128, 16, 96, 96, 2, 48, 0, seed=1)
    assert t2.reserve([0, 1], [500, 300]) == 0
    t2.append_all_layers([0, 1], [500, 300])
    used = sorted(c for r in (0, 1) for c in t2.o.table(r)[0].tolist() if c >= 0)
    free = sorted(set(range(96)) - set(used))
    assert t2.migrate(used[::-1][:10], free[:10]) == 0
    t2.check_bytes()
    t2.attention(1, [1, 0])


def case_pdl():
    import torch
    from tests.twin import Twin
    L, Hq, Hkv, d, T, R = 3, 32, 8, 128, 16, 4
    lens = [2900, 1700, 3333, 2047]  # >= 148 tiles: a full grid, where launch overlap is on
    MC = 4096 // T
    t = Twin(L, Hq, Hkv, d, T, R * MC, R * MC, R, MC, 0, seed=21)
    assert t.p.set_launch_overlap(True) == 0
    reqs = list(range(R))
    assert t.reserve(reqs, lens) == 0
    t.append_all_layers(reqs, lens)
    assert t.reserve(reqs, [1] * R) == 0
    for l in range(L):
        t.decode_fused(l, reqs)
    torch.cuda.synchronize()


def case_gather():
    import torch
    from paper_2506_15155_b200 import ellm, shard
    from inputs import workload as W
    from inputs.workload import Workload
    world, L, Hq, Hkv, d, B, ctx, T = 2, 2, 32, 8, 128, 3, 700, 16
    wls = [Workload("g", L, Hq, Hkv, d, B, ctx, 7, tokens_per_chunk=T * world, world=world, rank=i,
                    decode_headroom=64) for i in range(world)]
    pools = [W.make_pool(w, 0) for w in wls]
    for p, w in zip(pools, wls):
        W.prefill(p, w)
    nbytes = shard.gather_window_bytes(L, B, Hq, d)
    stride = shard.layer_stride(B, Hq, d)
    wins = [ellm.gather_window_create(0, nbytes)[0] for _ in range(world)]
    for i, p in enumerate(pools):
        assert p.gather_attach(world, i, Hq, wins, nbytes) == ellm.OK
    reqs = list(range(B))
    lens = np.full(B, ctx, np.int64)
    ins = [W.decode_inputs(w, 0, lens) for w in wls]
    for p in pools:
        assert p.reserve(reqs, [1] * B) == ellm.OK
    for l in range(L):
        for i, p in enumerate(pools):
            q, k, v = ins[i]
            if l > 0:
                assert p.gather_wait_next(l - 1) == ellm.OK
            assert p.attention_gather(l, reqs, q[l], l * stride, 1.0 / np.sqrt(d), k[l], v[l]) == ellm.OK
    for p in pools:
        assert p.gather_wait(L - 1) == ellm.OK
    torch.cuda.synchronize()
    for p in pools:
        p.gather_detach()
        p.close()
    for w in wins:
        ellm.gather_window_destroy(w)


def case_prefill():
    from tests.twin import Twin
    rng = np.random.default_rng(1)
    t = Twin(2, 32, 8, 128, 16, 160, 160, 2, 80, 0, seed=4, needle=False)
    assert t.reserve([0, 1], [700, 300]) == 0
    t.append_all_layers([0, 1], [700, 300])
    t.prefill(1, [0, 1], [300, 300], rng)


CASES = {"c1": case_c1, "pdl": case_pdl, "gather": case_gather, "prefill": case_prefill}

if __name__ == "__main__":
    import torch
    assert torch.cuda.is_available()
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print(f"case {name}: ok", flush=True)

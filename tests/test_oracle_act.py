"""Pins for the oracle's activation eTensor slots (O10/O11 in oracle.h) and
for grow's skipping of live slots (O9; "unmaps physical memory chunks allocated to
inactive eTensor objects"). Every expected value below is derived by hand from the written
policy (R15/R16): a slot is the run of consecutive idle ACT chunks with the highest last
id; grow takes the lowest idle ACT ids. A product-side twin on a host-only pool (no GPU) must
reach the same states.
"""
import numpy as np

import oracle
from oracle import Oracle

NO_CHUNKS, NOT_MAPPED, OUT_OF_RANGE, INVALID_ARG = -3, -6, -2, -1


def small(C, Ckv):
    # L=1, Hq=2, Hkv=1, d=64, T=16 (4 KiB chunks); 2 requests of up to 16 chunks
    return Oracle(1, 2, 1, 64, 16, C, Ckv, 2, 16, 4)


def test_slots_fill_from_the_top_and_grow_skips_them():
    o = small(16, 4)                       # KV 0..3, ACT 4..15
    assert o.act_alloc(3) == (0, 13)       # 13..15
    assert o.act_alloc(2) == (0, 11)       # 11..12
    assert o.act_alloc(0)[0] == INVALID_ARG
    s = o.stats()
    assert s["act"] == 12 and s["act_used"] == 5
    assert o.grow(8) == NO_CHUNKS          # idle ACT: 4..10 = 7 chunks
    assert o.grow(7) == 0                  # KV 0..10
    assert o.act_alloc(1)[0] == NO_CHUNKS  # no idle ACT left
    assert o.act_free(14) == NOT_MAPPED    # not a slot start
    assert o.act_free(16) == OUT_OF_RANGE
    assert o.act_free(13) == 0
    assert o.act_free(13) == NOT_MAPPED
    assert o.grow(3) == 0                  # 13, 14, 15 (11, 12 still hold activations)
    # the lowest-id reservation walks around the live slot: 0..10 then 13..15
    assert o.reserve([0], [14 * 16]) == 0
    assert o.table(0)[0].tolist() == list(range(11)) + [13, 14, 15]
    assert o.check_invariants() == 0
    s = o.stats()
    assert (s["kv_used"], s["kv_free"], s["act"], s["act_used"]) == (14, 0, 2, 2)


def test_fragmented_slots_take_the_highest_fitting_run():
    o = small(10, 0)
    assert o.act_alloc(2) == (0, 8)
    assert o.act_alloc(3) == (0, 5)
    assert o.act_alloc(2) == (0, 3)        # idle: 0..2
    assert o.act_free(5) == 0              # idle: 0..2, 5..7
    assert o.act_alloc(4)[0] == NO_CHUNKS  # two runs of 3
    assert o.act_alloc(3) == (0, 5)        # highest fitting run
    assert o.act_alloc(1) == (0, 2)
    assert o.stats()["act_used"] == 8      # slots 8..9, 5..7, 3..4, 2
    assert o.check_invariants() == 0


def test_shrink_returns_kv_chunks_that_slots_can_then_use():
    o = small(8, 8)                        # all KV
    assert o.act_alloc(1)[0] == NO_CHUNKS
    assert o.reserve([0], [3 * 16]) == 0   # 0..2 used
    assert o.shrink(5) == 0                # 3..7 -> ACT
    assert o.act_alloc(5) == (0, 3)
    assert o.grow(1) == NO_CHUNKS
    assert o.check_invariants() == 0


def test_random_ops_keep_invariants_and_match_host_only_pool():
    """Random reserve / release / grow / shrink / act_alloc / act_free on the oracle and on the
    product's host-metadata pool (ELLM_DEVICE_NONE): identical return codes, slot ids, tables
    and counters, and I1-I7 after every op."""
    from paper_2506_15155_b200 import ellm
    rng = np.random.default_rng(21)
    C, R = 48, 4
    o = Oracle(1, 2, 1, 64, 16, C, 12, R, 24, 8)
    p = ellm.Pool(ellm.DEVICE_NONE, 1, 2, 1, 64, 16, C, 12, R, 24, 8)
    slots = []
    for it in range(400):
        op = int(rng.integers(0, 6))
        if op == 0:
            r, n = int(rng.integers(0, R)), int(rng.integers(1, 80))
            assert o.reserve([r], [n]) == p.reserve([r], [n])
        elif op == 1:
            r = int(rng.integers(0, R))
            assert o.release(r) == p.release(r)
        elif op == 2:
            n = int(rng.integers(0, 10))
            assert o.grow(n) == p.grow(n)
        elif op == 3:
            n = int(rng.integers(0, 10))
            assert o.shrink(n) == p.shrink(n)
        elif op == 4:
            n = int(rng.integers(1, 8))
            a, b = o.act_alloc(n), p.act_alloc(n)
            assert a[0] == b[0] and (a[0] != 0 or a[1] == b[1]), (a, b)
            if a[0] == 0:
                slots.append(a[1])
        else:
            if slots and rng.random() < 0.8:
                first = slots.pop(int(rng.integers(0, len(slots))))
            else:
                first = int(rng.integers(0, C))
            assert o.act_free(first) == p.act_free(first)
        assert o.check_invariants() == 0
        so, sp = o.stats(), p.stats()
        assert all(so[k] == sp[k] for k in so), (so, sp)
        for r in range(R):
            assert o.table(r)[0].tolist() == p.table(r)[0].tolist()

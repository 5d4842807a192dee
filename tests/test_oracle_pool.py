"""Pins for the oracle's pool / page-table state machine (runs on CPU).

Closed forms from tests/golden/tables_c1.json, the chunk-layout golden
offsets (tests/golden/layout_c1.json), error conventions (include/ellm.h), and the
invariants I1-I6 checked after every operation of long random operation sequences.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import Oracle
from inputs import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def c1_oracle():
    g = json.load(open(os.path.join(GOLD, "tables_c1.json")))
    return Oracle(**g["config"]), g


def test_c1_chunk_bytes():
    o, g = c1_oracle()
    assert o.chunk_bytes == g["chunk_bytes"] == 8 * 1024


def test_chunk_arithmetic_llama8b():
    # S:46 128 KiB/token for LLaMA-3-8B; S:164 262144 tokens = 16384 chunks of 2 MiB
    o = Oracle(32, 32, 8, 128, 16, 4, 4, 1, 16384, 0)
    assert o.chunk_bytes == 2 * 1024 * 1024
    assert o.chunk_bytes // 16 == 128 * 1024
    assert 262144 * 128 * 1024 // o.chunk_bytes == 16384


def test_c1_tables_closed_form():
    o, g = c1_oracle()
    assert o.reserve([0, 1, 2, 3], g["prefill_lengths"]) == oracle.OK
    for r, want in enumerate(g["tables_after_prefill"]):
        t, ln = o.table(r)
        assert t.tolist() == want and ln == g["prefill_lengths"][r]
    assert o.reserve([0, 1, 2, 3], [1, 1, 1, 1]) == oracle.OK
    for r, want in enumerate(g["tables_after_one_decode"]):
        assert o.table(r)[0].tolist() == want
    assert o.stats() == {**g["stats_after_one_decode"], "act_used": 0}
    assert o.check_invariants() == 0


def _fill(o, g, seed=0):
    """Prefill C1 with generated K/V (layer 0) and return the per-request logical K/V."""
    L, Hkv, d = 1, 2, 64
    lens = g["prefill_lengths"]
    o.reserve([0, 1, 2, 3], lens)
    K, V = [], []
    for r, n in enumerate(lens):
        k, v = gen.request_kv(seed, r, n, 0, range(Hkv), d, 2, needle_range=n)
        K.append(k); V.append(v)
    assert o.append(0, [0, 1, 2, 3], lens, np.concatenate(K), np.concatenate(V)) == oracle.OK
    return K, V


def test_layout_golden_offsets():
    lay = json.load(open(os.path.join(GOLD, "layout_c1.json")))
    o, g = c1_oracle()
    K, V = _fill(o, g)
    # request 3 logical chunk 0 is chunk 15 (closed form); rows 0..15 are positions 0..15
    img = o.read_chunk(15)
    for c in lay["cases"]:
        src = (K if c["kv"] == 0 else V)[3][c["row"], c["head"], c["dim"]]
        got = int(img[c["byte"]]) | (int(img[c["byte"] + 1]) << 8)
        assert got == int(src), c


def test_deflate_inflate_closed_form_and_identity():
    o, g = c1_oracle()
    K, V = _fill(o, g)
    q = gen.q_bits(0, 3, 0, range(4), 64)[None]
    rc, before = o.attention(0, [3], q, 0.125)
    assert rc == oracle.OK
    imgs = [o.read_chunk(c) for c in g["deflate_r3_first8_chunk_ids"]]
    rc, slots = o.deflate(g["deflate_r3_first8_chunk_ids"])
    assert rc == oracle.OK and slots.tolist() == g["deflate_host_slots"]
    assert o.table(3)[0].tolist() == g["r3_table_after_deflate"]
    for h, img in zip(slots, imgs):
        assert np.array_equal(o.read_host_slot(h), img)
    assert o.attention(0, [3], q, 0.125)[0] == oracle.NOT_RESIDENT
    assert o.attention(0, [2], gen.q_bits(0, 2, 0, range(4), 64)[None], 0.125)[0] == oracle.OK
    assert o.check_invariants() == 0
    rc, ids = o.inflate(slots)
    assert rc == oracle.OK and ids.tolist() == g["inflate_chunk_ids"]
    assert o.table(3)[0].tolist() == g["tables_after_prefill"][3]
    rc, after = o.attention(0, [3], q, 0.125)
    assert rc == oracle.OK and np.array_equal(before, after)  # I5
    assert o.check_invariants() == 0


def test_through_table_equals_contiguous():
    o, g = c1_oracle()
    _fill(o, g)
    o.migrate([33, 5], [40, 50])
    o.deflate([0, 1])
    o.inflate([0, 1])
    q = np.stack([gen.q_bits(7, r, 0, range(4), 64) for r in range(4)])
    rc1, a = o.attention(0, [0, 1, 2, 3], q, 0.125, through_table=True)
    rc2, b = o.attention(0, [0, 1, 2, 3], q, 0.125, through_table=False)
    assert rc1 == rc2 == oracle.OK and np.array_equal(a, b)


def test_migrate_compaction_closed_form():
    o, g = c1_oracle()
    _fill(o, g)
    o.release(1)  # frees 2..5
    # compaction: highest USED ids -> lowest FREE ids
    assert o.migrate([33, 32, 31, 30], [2, 3, 4, 5]) == oracle.OK
    t3 = o.table(3)[0].tolist()
    assert t3[-4:] == [5, 4, 3, 2]
    assert o.stats()["kv_used"] == 30
    assert o.shrink(34) == oracle.OK          # ids 30..63 are FREE now: exactly 34
    assert o.stats() == {"kv_free": 0, "kv_used": 30, "act": 34, "host_free": 64, "host_used": 0, "act_used": 0}
    assert o.shrink(1) == oracle.IN_USE
    assert o.grow(2) == oracle.OK             # lowest ACT ids: 30, 31
    assert o.reserve([1], [20]) == oracle.OK
    assert o.table(1)[0].tolist() == [30, 31]
    assert o.check_invariants() == 0


def test_error_codes():
    o, g = c1_oracle()
    _fill(o, g)
    assert o.reserve([4], [1]) == oracle.OUT_OF_RANGE
    assert o.reserve([0, 0], [1, 1]) == oracle.INVALID_ARG
    assert o.reserve([0], [-1]) == oracle.INVALID_ARG
    assert o.reserve([0], [16 * 32]) == oracle.OUT_OF_RANGE      # > max_chunks_per_request
    assert o.reserve([0, 1], [16 * 20, 16 * 20]) == oracle.NO_CHUNKS
    assert o.stats()["kv_used"] == 34                             # all-or-nothing
    assert o.append(1, [0], [17], np.zeros((17, 2, 64)), np.zeros((17, 2, 64))) == oracle.OUT_OF_RANGE
    assert o.append(0, [0], [3], np.zeros((3, 2, 64)), np.zeros((3, 2, 64))) == oracle.INVALID_ARG
    assert o.deflate([63])[0] == oracle.NOT_MAPPED
    assert o.deflate([64])[0] == oracle.OUT_OF_RANGE
    assert o.deflate([1, 1])[0] == oracle.INVALID_ARG
    assert o.inflate([0])[0] == oracle.NOT_MAPPED
    assert o.migrate([0], [1]) == oracle.ALREADY_MAPPED
    assert o.migrate([40], [41]) == oracle.NOT_MAPPED
    assert o.migrate([0], [0]) == oracle.INVALID_ARG
    o.release(0)
    assert o.attention(0, [0], np.zeros((1, 4, 64), np.uint16), 1.0)[0] == oracle.INVALID_ARG
    # partially filled last chunk on HOST -> cannot reserve into it
    o.reserve([0], [5])
    o.deflate([o.table(0)[0][0]])
    assert o.reserve([0], [1]) == oracle.NOT_RESIDENT
    assert o.check_invariants() == 0
    small = Oracle(1, 1, 1, 8, 4, 8, 8, 2, 8, 1)
    small.reserve([0], [12])
    assert small.deflate([0, 1])[0] == oracle.HOST_FULL
    assert small.grow(1) == oracle.NO_CHUNKS


def _random_ops(seed, n_ops):
    rng = np.random.default_rng(seed)
    L, Hq, Hkv, d, T = 2, 4, 2, 8, 4
    C, H, R, MC = 48, 16, 6, 10
    o = Oracle(L, Hq, Hkv, d, T, C, 32, R, MC, H)
    counts = {}
    for _ in range(n_ops):
        op = rng.integers(0, 8)
        if op in (0, 1):
            reqs = rng.choice(R, size=rng.integers(1, 4), replace=False)
            nn = rng.integers(0, 9, size=len(reqs))
            rc = o.reserve(reqs, nn)
            if rc == oracle.OK:
                for l in range(L):
                    rows = int(nn.sum())
                    kb = rng.integers(0, 1 << 16, size=(rows, Hkv, d), dtype=np.uint16)
                    vb = rng.integers(0, 1 << 16, size=(rows, Hkv, d), dtype=np.uint16)
                    rc2 = o.append(l, reqs, nn, kb, vb)
                    assert rc2 in (oracle.OK, oracle.NOT_RESIDENT)
        elif op == 2:
            used = [c for r in range(R) for c in o.table(r)[0].tolist() if c >= 0]
            if used:
                ids = rng.choice(used, size=min(len(used), rng.integers(1, 4)), replace=False)
                rc, _ = o.deflate(ids)
        elif op == 3:
            hs = [-e - 2 for r in range(R) for e in o.table(r)[0].tolist() if e <= -2]
            if hs:
                sl = rng.choice(hs, size=min(len(hs), rng.integers(1, 4)), replace=False)
                rc, _ = o.inflate(sl)
        elif op == 4:
            used = [c for r in range(R) for c in o.table(r)[0].tolist() if c >= 0]
            st = o.stats()
            free = [c for c in range(C) if c not in used][: st["kv_free"]]
            if used:
                src = rng.choice(used, size=1)
                dst = rng.choice(range(C), size=1)
                rc = o.migrate(src, dst)
        elif op == 5:
            rc = o.release(int(rng.integers(0, R)))
        elif op == 6:
            rc = o.grow(int(rng.integers(0, 4)))
        else:
            rc = o.shrink(int(rng.integers(0, 4)))
        counts[op] = counts.get(op, 0) + 1
        inv = o.check_invariants()
        assert inv == 0, f"invariant I{inv} violated after op {op}"
    return counts


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_random_sequences_keep_invariants(seed):
    counts = _random_ops(seed, 2500)
    assert len(counts) == 8

"""Host logic of libellm.so (allocation, tables, ownership, host slots, error codes) against
the oracle, on a host-metadata-only pool (device = ELLM_DEVICE_NONE; no GPU needed).
Tables, stats and every status code must be identical (bit-exact integer state)."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import Oracle
from paper_2506_15155_b200 import ellm

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def pair(L=2, Hq=4, Hkv=2, d=64, T=16, C=48, Ckv=32, R=6, MC=10, H=16):
    o = Oracle(L, Hq, Hkv, d, T, C, Ckv, R, MC, H)
    p = ellm.Pool(ellm.DEVICE_NONE, L, Hq, Hkv, d, T, C, Ckv, R, MC, H)
    return o, p


def same_state(o, p, R):
    for r in range(R):
        to, lo = o.table(r)
        tp, lp = p.table(r)
        assert lo == lp and to.tolist() == tp.tolist(), (r, to, tp)
    so, sp = o.stats(), p.stats()
    for k in so:
        assert so[k] == sp[k], (k, so, sp)


def test_c1_closed_form_matches():
    g = json.load(open(os.path.join(GOLD, "tables_c1.json")))
    c = g["config"]
    p = ellm.Pool(ellm.DEVICE_NONE, c["n_layers"], c["n_heads_q"], c["n_heads_kv"], c["head_dim"],
                  c["tokens_per_chunk"], c["max_chunks"], c["initial_chunks"], c["max_requests"],
                  c["max_chunks_per_request"], c["host_slots"])
    assert p.chunk_bytes == g["chunk_bytes"]
    assert p.reserve([0, 1, 2, 3], g["prefill_lengths"]) == 0
    assert [p.table(r)[0].tolist() for r in range(4)] == g["tables_after_prefill"]
    assert p.reserve([0, 1, 2, 3], [1, 1, 1, 1]) == 0
    assert [p.table(r)[0].tolist() for r in range(4)] == g["tables_after_one_decode"]
    rc, slots = p.deflate(g["deflate_r3_first8_chunk_ids"])
    assert rc == 0 and slots.tolist() == g["deflate_host_slots"]
    assert p.table(3)[0].tolist() == g["r3_table_after_deflate"]
    assert p.attention(0, [3], 0, 0, 1.0) == ellm.NOT_RESIDENT
    rc, ids = p.inflate(slots)
    assert rc == 0 and ids.tolist() == g["inflate_chunk_ids"]


@pytest.mark.parametrize("seed", range(6))
def test_random_ops_match_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    L, Hq, Hkv, d, T, C, Ckv, R, MC, H = 2, 4, 2, 64, 16, 48, 32, 6, 10, 16
    o, p = pair(L, Hq, Hkv, d, T, C, Ckv, R, MC, H)
    seen = set()
    for step in range(800):
        op = int(rng.integers(0, 9))
        if op <= 1:
            reqs = rng.choice(R + 1, size=int(rng.integers(1, 4)), replace=bool(rng.integers(0, 8) == 0))
            nn = rng.integers(-1 if rng.integers(0, 20) == 0 else 0, 40, size=len(reqs))
            a, b = o.reserve(reqs, nn), p.reserve(reqs, nn)
        elif op == 2:
            reqs = rng.choice(R + 1, size=int(rng.integers(1, 3)), replace=False)
            nn = [int(x) for x in rng.integers(0, 3, size=len(reqs))]
            rows = max(sum(nn), 1)
            a = o.append(int(rng.integers(0, L + 1)) if rng.integers(0, 10) == 0 else 0, reqs, nn,
                         np.zeros((rows, Hkv, d), np.uint16), np.zeros((rows, Hkv, d), np.uint16))
            b = p.append(0 if a != oracle.OUT_OF_RANGE else L, reqs, nn, 0, 0)
            if a == oracle.OK:
                a = ellm.NO_DEVICE
        elif op == 3:
            ids = rng.integers(-1, C + 1, size=int(rng.integers(1, 4)))
            (a, sa), (b, sb) = o.deflate(ids), p.deflate(ids)
            if a == 0:
                assert sa.tolist() == sb.tolist()
        elif op == 4:
            sl = rng.integers(-1, H + 1, size=int(rng.integers(1, 4)))
            (a, ia), (b, ib) = o.inflate(sl), p.inflate(sl)
            if a == 0:
                assert ia.tolist() == ib.tolist()
        elif op == 5:
            n = int(rng.integers(1, 3))
            src, dst = rng.integers(0, C, size=n), rng.integers(0, C, size=n)
            a, b = o.migrate(src, dst), p.migrate(src, dst)
        elif op == 6:
            r = int(rng.integers(-1, R + 1))
            a, b = o.release(r), p.release(r)
        elif op == 7:
            n = int(rng.integers(-1, 5))
            a, b = o.grow(n), p.grow(n)
        else:
            n = int(rng.integers(-1, 5))
            a, b = o.shrink(n), p.shrink(n)
        assert a == b, (step, op, a, b)
        seen.add((op, a))
        same_state(o, p, R)
    assert len({a for _, a in seen}) >= 5  # several distinct status codes exercised


def test_deflate_slot_ids_match_oracle():
    o, p = pair()
    for x in (o, p):
        assert x.reserve([0, 1, 2], [40, 17, 33]) == 0
    ids = [5, 0, 3, 7]
    (a, sa), (b, sb) = o.deflate(ids), p.deflate(ids)
    assert a == b == 0 and sa.tolist() == sb.tolist() == [0, 1, 2, 3]
    (a, sa), (b, sb) = o.inflate([2, 0]), p.inflate([2, 0])
    assert a == b == 0 and sa.tolist() == sb.tolist()
    same_state(o, p, 6)

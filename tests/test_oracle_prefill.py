"""Pins for the oracle's chunked-prefill attention (O12).

The stateful oracle is filled through reserve / append and its causal prefill output is
compared with numpy brute force (oracle/brute.py: an explicit lower-triangular mask on the
score matrix, written with array primitives) on the same bf16 inputs, plus closed forms:
the query at position 0 returns v_0 exactly; a single query at the last position equals the
decode attention (O4); table and contiguous reads agree exactly.
"""
import numpy as np
import pytest

from oracle import Oracle, brute
from inputs import gen

RNG = np.random.default_rng(77)


def rand_bits(shape):
    return gen.f32_to_bf16(RNG.standard_normal(shape).astype(np.float32))


def filled(L, Hq, Hkv, d, T, lens, C=64):
    o = Oracle(L, Hq, Hkv, d, T, C, C, len(lens), C, 8)
    assert o.reserve(list(range(len(lens))), lens) == 0
    kv = {}
    for r, n in enumerate(lens):
        for l in range(L):
            k, v = rand_bits((n, Hkv, d)), rand_bits((n, Hkv, d))
            assert o.append(l, [r], [n], k, v) == 0
            kv[(r, l)] = (k, v)
    return o, kv


@pytest.mark.parametrize("Hq,Hkv,d,T,lens,nq", [
    (4, 2, 64, 16, [50, 17], [20, 17]),
    (8, 2, 128, 32, [130, 5, 64], [130, 1, 33]),
    (4, 4, 32, 16, [40], [7]),
])
def test_matches_numpy_causal_bruteforce(Hq, Hkv, d, T, lens, nq):
    o, kv = filled(2, Hq, Hkv, d, T, lens)
    q = rand_bits((sum(nq), Hq, d))
    scale = 1.0 / np.sqrt(d)
    for l in range(2):
        rc, out = o.prefill_attention(l, list(range(len(lens))), nq, q, scale)
        assert rc == 0
        row = 0
        for r, (n, m) in enumerate(zip(lens, nq)):
            k, v = kv[(r, l)]
            ref = brute.causal_prefill(q[row:row + m], k, v, scale)
            np.testing.assert_allclose(out[row:row + m], ref, rtol=1e-12, atol=1e-13)
            row += m
        rc2, out2 = o.prefill_attention(l, list(range(len(lens))), nq, q, scale, through_table=False)
        assert rc2 == 0 and np.array_equal(out, out2)


def test_position_zero_returns_v0_and_last_query_equals_decode():
    o, kv = filled(1, 4, 2, 64, 16, [33])
    q = rand_bits((33, 4, 64))
    rc, out = o.prefill_attention(0, [0], [33], q, 0.125)
    assert rc == 0
    v0 = brute.bf16_bits_to_f64(kv[(0, 0)][1][0])
    for h in range(4):
        assert np.array_equal(out[0, h], v0[h // 2])
    rc, dec = o.attention(0, [0], q[32:33], 0.125)
    assert rc == 0 and np.array_equal(out[32], dec[0])


def test_prefill_errors():
    o, _ = filled(1, 4, 2, 64, 16, [20, 5])
    q = rand_bits((30, 4, 64))
    assert o.prefill_attention(1, [0], [1], q, 0.1)[0] == -2          # layer range
    assert o.prefill_attention(0, [2], [1], q, 0.1)[0] == -2          # request range
    assert o.prefill_attention(0, [0], [0], q, 0.1)[0] == -1          # n_q < 1
    assert o.prefill_attention(0, [1], [6], q, 0.1)[0] == -1          # n_q > len
    rc, slots = o.deflate([int(o.table(1)[0][0])])
    assert rc == 0
    assert o.prefill_attention(0, [0, 1], [3, 3], q, 0.1)[0] == -5    # not resident

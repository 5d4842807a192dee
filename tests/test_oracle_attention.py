"""Pins for the oracle's attention arithmetic (runs on CPU).

The oracle (oracle/oracle.cpp, fp64 loops) is checked against things other than itself:
numpy brute force written with array primitives (oracle/brute.py), closed-form special
cases, and invariances that the softmax-attention definition fixes.
"""
import numpy as np
import pytest

import oracle
from oracle import brute
from inputs import gen

RNG = np.random.default_rng(1234)


def rand_bits(shape, scale=1.0):
    return gen.f32_to_bf16(RNG.standard_normal(shape).astype(np.float32) * np.float32(scale))


@pytest.mark.parametrize("Hq,Hkv,d,n", [(4, 2, 64, 17), (4, 2, 64, 300), (8, 8, 32, 5),
                                        (32, 8, 128, 129), (64, 8, 128, 40), (6, 2, 16, 1)])
def test_matches_numpy_bruteforce(Hq, Hkv, d, n):
    q, k, v = rand_bits((Hq, d)), rand_bits((n, Hkv, d)), rand_bits((n, Hkv, d))
    scale = 1.0 / np.sqrt(d)
    o = oracle.attention_contig(q, k, v, scale)
    ref = brute.attention(q, k, v, scale)
    np.testing.assert_allclose(o, ref, rtol=1e-12, atol=1e-13)


def test_len1_returns_v0_exactly():
    q, k, v = rand_bits((4, 64)), rand_bits((1, 2, 64)), rand_bits((1, 2, 64))
    o = oracle.attention_contig(q, k, v, 0.125)
    vv = brute.bf16_bits_to_f64(v)
    for h in range(4):
        assert np.array_equal(o[h], vv[0, h // 2])


def test_equal_keys_give_mean_of_v():
    n = 37
    k = np.repeat(rand_bits((1, 2, 64)), n, axis=0)
    q, v = rand_bits((4, 64)), rand_bits((n, 2, 64))
    o = oracle.attention_contig(q, k, v, 0.125)
    mean = brute.bf16_bits_to_f64(v).mean(axis=0)
    for h in range(4):
        np.testing.assert_allclose(o[h], mean[h // 2], rtol=1e-13, atol=1e-14)


def test_constant_v_rows_returned_exactly():
    n = 50
    v = np.repeat(rand_bits((1, 2, 64)), n, axis=0)
    q, k = rand_bits((4, 64)), rand_bits((n, 2, 64))
    o = oracle.attention_contig(q, k, v, 0.125)
    vv = brute.bf16_bits_to_f64(v)
    for h in range(4):
        np.testing.assert_allclose(o[h], vv[0, h // 2], rtol=1e-14, atol=0)


def test_needle_dominates():
    """A key with logit gap >= 40 over all others returns its value row to fp64 precision."""
    d, n = 64, 200
    q = np.zeros((1, d), np.uint16)
    q[0, 0] = gen.f32_to_bf16(np.float32(1.0))
    k = np.zeros((n, 1, d), np.uint16)
    k[77, 0, 0] = gen.f32_to_bf16(np.float32(64.0))  # s = 64 * 1 * scale(1) vs 0 elsewhere
    v = rand_bits((n, 1, d))
    o = oracle.attention_contig(q, k, v, 1.0)
    # every other weight is e^-64 / (1 + ...) < 1e-27: the result is v_77 to fp64 precision
    np.testing.assert_allclose(o[0], brute.bf16_bits_to_f64(v)[77, 0], rtol=1e-15, atol=1e-25)


def test_mha_equals_per_head_single_head_attention():
    Hq = Hkv = 4
    d, n = 32, 33
    q, k, v = rand_bits((Hq, d)), rand_bits((n, Hkv, d)), rand_bits((n, Hkv, d))
    o = oracle.attention_contig(q, k, v, 0.2)
    for h in range(Hq):
        oh = oracle.attention_contig(q[h:h + 1], k[:, h:h + 1], v[:, h:h + 1], 0.2)
        assert np.array_equal(o[h], oh[0])


def test_head_permutation_within_group_permutes_output():
    Hq, Hkv, d, n = 8, 2, 32, 21
    q, k, v = rand_bits((Hq, d)), rand_bits((n, Hkv, d)), rand_bits((n, Hkv, d))
    o = oracle.attention_contig(q, k, v, 0.3)
    perm = np.array([3, 2, 1, 0, 5, 7, 4, 6])  # permutes within each group of 4
    op = oracle.attention_contig(q[perm], k, v, 0.3)
    assert np.array_equal(op, o[perm])


def test_gqa_head_to_kv_mapping_is_contiguous_groups():
    """q-head h must read kv-head h // group: zero all kv-heads but one and check which
    q-heads see it (a transposed or modulo mapping fails)."""
    Hq, Hkv, d, n = 8, 4, 16, 9
    q = rand_bits((Hq, d))
    k = rand_bits((n, Hkv, d))
    v = np.zeros((n, Hkv, d), np.uint16)
    v[:, 1, :] = gen.f32_to_bf16(np.float32(1.0))
    o = oracle.attention_contig(q, k, v, 0.25)
    for h in range(Hq):
        expect = 1.0 if h // 2 == 1 else 0.0
        assert np.all(o[h] == expect)


def test_shift_invariance_and_scale_matters():
    Hq, Hkv, d, n = 2, 1, 16, 12
    q, k, v = rand_bits((Hq, d)), rand_bits((n, Hkv, d)), rand_bits((n, Hkv, d))
    a = oracle.attention_contig(q, k, v, 0.5)
    b = oracle.attention_contig(q, k, v, 0.25)
    assert not np.allclose(a, b)
    np.testing.assert_allclose(a, brute.attention(q, k, v, 0.5), rtol=1e-12, atol=1e-13)


def test_bad_args():
    with pytest.raises(ValueError):
        oracle.attention_contig(np.zeros((3, 8), np.uint16), np.zeros((4, 2, 8), np.uint16),
                                np.zeros((4, 2, 8), np.uint16), 1.0)

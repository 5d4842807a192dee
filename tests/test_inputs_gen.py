"""Pins for the seeded input generator (inputs/gen.py): splitmix64 reference outputs,
RNE rounding, distribution, needles. The CUDA twin (inputs/gen.cu) is pinned against
this in tests/test_gpu_parity.py."""
import json
import os

import numpy as np

from inputs import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_values():
    g = json.load(open(os.path.join(GOLD, "splitmix64.json")))
    gamma = int(gen.GOLDEN)
    for i, want in enumerate(g["state0_outputs"]):
        assert int(gen.splitmix64(np.uint64((i * gamma) % 2 ** 64))) == int(want, 16)


def test_rne_rounding():
    x = np.array([1.0, 1.00390625, 1.01171875, -1.00390625, 0.0, 3.0], np.float32)
    # 1+2^-8 is a tie -> even (1.0); 1+3*2^-8 tie -> even (1+2^-6... = 0x3F82)
    assert gen.f32_to_bf16(x).tolist() == [0x3F80, 0x3F80, 0x3F82, 0xBF80, 0, 0x4040]


def test_distribution_and_determinism():
    b = gen.bf16_from_hash(gen.hash_at(5, gen.STREAM_K, np.arange(200000)))
    f = gen.bf16_to_f32(b)
    assert abs(f.mean()) < 0.01 and abs(f.std() - 1.1547) < 0.01
    assert np.array_equal(b, gen.bf16_from_hash(gen.hash_at(5, gen.STREAM_K, np.arange(200000))))
    assert not np.array_equal(b, gen.bf16_from_hash(gen.hash_at(6, gen.STREAM_K, np.arange(200000))))


def test_needles():
    seed, r, l, d, group = 3, 2, 1, 64, 4
    k, v = gen.request_kv(seed, r, 100, l, [0, 1], d, group, needle_range=100)
    for h in (0, 1):
        pos = gen.needle_positions(seed, r, l, h, 100)
        assert len(pos) == 3 and np.all((pos >= 0) & (pos < 100))
        q0 = gen.bf16_to_f32(gen.q_bits(seed, r, l, [h * group], d)[0])
        for p in pos:
            assert np.array_equal(gen.bf16_to_f32(k[p, h]), 4 * q0)
            assert set(np.abs(gen.bf16_to_f32(v[p, h])).tolist()) == {3.0}


def test_sharded_heads_draw_same_values():
    k_all, _ = gen.request_kv(1, 0, 40, 0, range(8), 128, 4, needle_range=40)
    k_sh, _ = gen.request_kv(1, 0, 40, 0, range(4, 6), 128, 4, needle_range=40)
    assert np.array_equal(k_all[:, 4:6], k_sh)


def test_c5_length_mix_recipe():
    """BASELINE.json configs[4] length mix (inputs/c5.py): prompts log-uniform in [2K, 128K],
    outputs uniform in [16, 256], deterministic per seed."""
    import numpy as np
    from inputs.c5 import c5_lengths
    p, o = c5_lengths(256, 5)
    p2, o2 = c5_lengths(256, 5)
    assert np.array_equal(p, p2) and np.array_equal(o, o2)
    assert p.min() >= 2048 and p.max() <= 131072 and o.min() >= 16 and o.max() <= 256
    # log-uniform: log2 of the prompts is ~uniform on [11, 17]; mean of a log-uniform on
    # [a, b] is (b - a) / ln(b / a) = 30.5K
    lg = np.log2(p)
    assert abs(lg.mean() - 14.0) < 0.35
    assert 24000 < p.mean() < 37000
    assert not np.array_equal(c5_lengths(256, 6)[0], p)

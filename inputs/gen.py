"""Seeded synthetic input generator shared by tests, bench and oracle legs.

Holds NONE of the method's arithmetic: it only draws the K/V/Q values the method is
fed. Both sides get their inputs from here (numpy) or from ``inputs/gen.cu`` (the same
counter-based generator, bit-identical, for inputs too large to make on the host).

Counter-based generator:
    h   = splitmix64(splitmix64(seed ^ stream*C) + index)          (uint64, wraps)
    s   = sum of the four 16-bit lanes of h                          (Irwin-Hall, ~normal)
    f32 = float32(s - 131070) * 2**-15                                (exact; std ~1.155)
    bf16 = round-to-nearest-even of f32's top 16 bits                 (integer ops)
Every step is integer or exact, so numpy and CUDA produce identical bits.

Needles (SURVEY §8(d) "Synthetic inputs"): 3 positions per (request, layer, kv-head),
drawn in [0, needle_range). At a needle, K = 4 * q_{h0} (h0 = first q-head of the
group; *4 is exact in bf16) so head h0 puts a logit gap of ~4*sqrt(d) on it, and
V = +-3 per element. A wrong-chunk read then moves the output by O(1).

Index radices: request < 2**12, position < 2**21, layer < 2**8, head < 2**8, dim < 2**10.
Head indices are GLOBAL head ids, so a KV-head-sharded run draws exactly the same
values for its heads as the unsharded run.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)
STREAM_K, STREAM_V, STREAM_Q, STREAM_NEEDLE_POS, STREAM_NEEDLE_SIGN = 1, 2, 3, 4, 5
N_NEEDLES = 3
BF16_POS3, BF16_NEG3 = 0x4040, 0xC040


def splitmix64(z):
    """splitmix64 finaliser applied to state z (adds the golden gamma first)."""
    with np.errstate(over="ignore"):
        z = np.asarray(z, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return splitmix64(np.uint64(seed) ^ (np.uint64(stream) * STREAM_MUL))


def hash_at(seed: int, stream: int, index) -> np.ndarray:
    with np.errstate(over="ignore"):
        return splitmix64(stream_key(seed, stream) + np.asarray(index, dtype=np.uint64))


def bf16_from_hash(h: np.ndarray) -> np.ndarray:
    h = np.asarray(h, dtype=np.uint64)
    s = np.zeros(h.shape, dtype=np.int64)
    for i in range(4):
        s += ((h >> np.uint64(16 * i)) & np.uint64(0xFFFF)).astype(np.int64)
    f = (s - 131070).astype(np.float32) * np.float32(2.0 ** -15)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return u.astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bits (finite inputs)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return u.astype(np.uint16)


def _kv_index(r, p, l, h, e):
    r, p, l, h, e = (np.asarray(x, dtype=np.uint64) for x in (r, p, l, h, e))
    return (((((r << np.uint64(21)) | p) << np.uint64(8) | l) << np.uint64(8) | h) << np.uint64(10)) | e


def _q_index(r, l, h, e):
    r, l, h, e = (np.asarray(x, dtype=np.uint64) for x in (r, l, h, e))
    return (((r << np.uint64(8) | l) << np.uint64(8) | h) << np.uint64(10)) | e


def q_bits(seed: int, r: int, l: int, heads, d: int) -> np.ndarray:
    """Q for request r, layer l, global q-heads `heads` -> [len(heads), d] bf16 bits."""
    heads = np.asarray(heads, dtype=np.int64)
    idx = _q_index(r, l, heads[:, None], np.arange(d)[None, :])
    return bf16_from_hash(hash_at(seed, STREAM_Q, idx))


def needle_positions(seed: int, r: int, l: int, kv_head: int, needle_range: int) -> np.ndarray:
    """The N_NEEDLES needle positions of (r, l, kv_head), each in [0, needle_range)."""
    if needle_range <= 0:
        return np.zeros(0, dtype=np.int64)
    i = np.arange(N_NEEDLES, dtype=np.uint64)
    idx = (((np.uint64(r) << np.uint64(8) | np.uint64(l)) << np.uint64(8) | np.uint64(kv_head))
           << np.uint64(2)) | i
    return (hash_at(seed, STREAM_NEEDLE_POS, idx) % np.uint64(needle_range)).astype(np.int64)


def kv_bits(seed: int, r: int, positions, l: int, kv: int, heads, d: int, group: int,
            needle_range: int = 0) -> np.ndarray:
    """K (kv=0) or V (kv=1) rows for request r, layer l, at `positions`, global kv-heads
    `heads` -> [len(positions), len(heads), d] bf16 bits, needles applied."""
    pos = np.asarray(positions, dtype=np.int64)
    heads = np.asarray(heads, dtype=np.int64)
    e = np.arange(d)
    idx = _kv_index(r, pos[:, None, None], l, heads[None, :, None], e[None, None, :])
    out = bf16_from_hash(hash_at(seed, STREAM_K if kv == 0 else STREAM_V, idx))
    if needle_range > 0:
        for hi, h in enumerate(heads.tolist()):
            npos = needle_positions(seed, r, l, h, needle_range)
            hit = np.isin(pos, npos)
            if not hit.any():
                continue
            if kv == 0:
                q0 = q_bits(seed, r, l, [h * group], d)[0]
                k4 = np.where((q0 & 0x7FFF) == 0, q0, (q0.astype(np.uint32) + 0x0100).astype(np.uint16))
                out[hit, hi, :] = k4[None, :]
            else:
                sidx = idx[hit, hi, :]
                sign = hash_at(seed, STREAM_NEEDLE_SIGN, sidx) & np.uint64(1)
                out[hit, hi, :] = np.where(sign == 1, BF16_NEG3, BF16_POS3).astype(np.uint16)
    return out


def request_kv(seed: int, r: int, length: int, l: int, heads, d: int, group: int,
               needle_range: int = 0):
    """(K, V) for positions [0, length) -> two [length, len(heads), d] arrays."""
    pos = np.arange(length)
    return (kv_bits(seed, r, pos, l, 0, heads, d, group, needle_range),
            kv_bits(seed, r, pos, l, 1, heads, d, group, needle_range))

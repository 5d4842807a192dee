"""numpy brute-force textbook attention — the pin for the C++ oracle's arithmetic.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definition followed (causal attention over the accumulated KV; the decode
token attends to every cached position, reading R5):
    s_j = scale * <q_h, k_{j, g(h)}>,   g(h) = h // (Hq // Hkv)         (reading R6)
    o_h = sum_j softmax(s)_j v_{j, g(h)}
written with numpy array primitives (einsum / exp / sum) in float64, independently of
oracle.cpp's loops.
"""
from __future__ import annotations

import numpy as np


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> float64 (exact: bf16 is the top half of an fp32)."""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32).astype(np.float64)


def attention(q_bits: np.ndarray, k_bits: np.ndarray, v_bits: np.ndarray, scale: float) -> np.ndarray:
    """q_bits [Hq, d]; k_bits/v_bits [len, Hkv, d] (bf16 bits). Returns [Hq, d] float64."""
    q = bf16_bits_to_f64(q_bits)
    k = bf16_bits_to_f64(k_bits)
    v = bf16_bits_to_f64(v_bits)
    Hq = q.shape[0]
    Hkv = k.shape[1]
    group = Hq // Hkv
    k_full = np.repeat(k, group, axis=1)          # [len, Hq, d]
    v_full = np.repeat(v, group, axis=1)
    s = scale * np.einsum("hd,jhd->hj", q, k_full)  # [Hq, len]
    s = s - s.max(axis=1, keepdims=True)
    w = np.exp(s)
    w = w / w.sum(axis=1, keepdims=True)
    return np.einsum("hj,jhd->hd", w, v_full)


def causal_prefill(q_bits: np.ndarray, k_bits: np.ndarray, v_bits: np.ndarray, scale: float) -> np.ndarray:
    """Causal attention of the LAST nq positions of a sequence (f4).

    q_bits [nq, Hq, d]; k_bits/v_bits [len, Hkv, d]. Query i sits at position len - nq + i and
    sees keys 0..that position: a lower-triangular mask on the [nq, len] score matrix.
    Returns [nq, Hq, d] float64."""
    q = bf16_bits_to_f64(q_bits)
    k = bf16_bits_to_f64(k_bits)
    v = bf16_bits_to_f64(v_bits)
    nq, Hq, _ = q.shape
    n = k.shape[0]
    group = Hq // k.shape[1]
    k_full = np.repeat(k, group, axis=1)                      # [len, Hq, d]
    v_full = np.repeat(v, group, axis=1)
    s = scale * np.einsum("ihd,jhd->hij", q, k_full)            # [Hq, nq, len]
    pos = np.arange(nq)[:, None] + (n - nq)
    s = np.where(np.arange(n)[None, :] <= pos, s, -np.inf)
    s = s - s.max(axis=2, keepdims=True)
    w = np.exp(s)
    w = w / w.sum(axis=2, keepdims=True)
    return np.einsum("hij,jhd->ihd", w, v_full)

"""The FMA-pipe exp2 that prefill.cu (f4) uses for part of the softmax exponentials (ex2_fma2, a
pair at a time), emulated in float32 numpy step by step (round-to-nearest split by the 1.5*2^23
constant, x - (r - M), cubic in the fraction, exponent add), against numpy's exp2 in float64: relative error < 1e-4 over the range the
softmax feeds it (x <= 8 by the lazy-rescale headroom; clamped below at -125)."""
import re
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _coeffs():
    src = open(os.path.join(ROOT, "paper_2506_15155_b200", "csrc", "prefill.cu")).read()
    m = re.search(r"kE2C3 = ([-0-9.e]+)f, kE2C2 = ([-0-9.e]+)f, kE2C1 = ([-0-9.e]+)f, kE2C0 = ([-0-9.e]+)f", src)
    return [np.float32(float(v)) for v in m.groups()]


def ex2_fma(x):
    c3, c2, c1, c0 = _coeffs()
    x = np.maximum(x.astype(np.float32), np.float32(-125))
    r = (x + np.float32(12582912)).astype(np.float32)
    f = (x - (r - np.float32(12582912))).astype(np.float32)
    fma = lambda a, b, c: (a.astype(np.float64) * b.astype(np.float64) + np.float64(c)).astype(np.float32)  # noqa: E731
    q = fma(np.full_like(f, c3), f, c2)   # one rounding per step, as fma.rn.f32x2
    q = fma(q, f, c1)
    q = fma(q, f, c0)
    return (q.view(np.int32) + (r.view(np.int32) << 23)).astype(np.int32).view(np.float32)


def test_ex2_fma_relative_error():
    x = np.linspace(-124.9, 8.5, 1_000_001).astype(np.float32)
    y = ex2_fma(x).astype(np.float64)
    ref = np.exp2(x.astype(np.float64))
    assert np.max(np.abs(y - ref) / ref) < 1e-4


def test_ex2_fma_masked_scores_are_tiny_and_normal():
    y = ex2_fma(np.array([-np.inf, -1e30, -200.0], np.float32))
    assert np.all(y > 0) and np.all(y < 1e-37) and np.all(np.isfinite(y))

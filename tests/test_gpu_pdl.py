"""Programmatic dependent launch of the attention kernel (attention.cu, pool.cpp attention_impl):
consecutive attention launches on one stream overlap (the next one streams its layer's K/V
before griddepcontrol.wait). These tests issue long back-to-back sequences with NO host sync
in between — fused decode steps over all layers, and plain attention in orders that repeat a
layer right after a fused append into it (where PDL must be off) — and only then compare every
output with the oracle, which replays the same sequence. Sizes give full grids (one CTA per SM),
the configuration in which PDL is enabled."""
from __future__ import annotations

import numpy as np
import pytest

from tests.twin import Twin, bits_to_torch, check_attention, torch_to_bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pdl", ["1", "0"])
def test_back_to_back_attention_sequences(pdl, monkeypatch):
    monkeypatch.setenv("ELLM_PDL", pdl)
    L, Hq, Hkv, d, T = 4, 32, 8, 128, 16
    R = 4
    lens = [2900, 1700, 3333, 2047]          # >= 148 tiles of 16 tokens: a full grid
    MC = 4096 // T
    C = R * MC
    t = Twin(L, Hq, Hkv, d, T, C, C, R, MC, 0, seed=21)
    assert t.p.set_launch_overlap(True) == 0   # the environment (ELLM_PDL) wins over it
    reqs = list(range(R))
    assert t.reserve(reqs, lens) == 0
    t.append_all_layers(reqs, lens)
    # decode steps: reserve +1 then fused append + attention per layer, back to back
    for step in range(2):
        assert t.reserve(reqs, [1] * R) == 0
        _run_fused_step(t, reqs)
    # plain attention, including the same layer right after a fused append into it
    assert t.reserve(reqs, [1] * R) == 0
    _run_mixed(t, reqs)


def _run_fused_step(t, reqs):
    import torch
    staged, outs = [], []
    for layer in range(t.L):
        q = t.q_bits(reqs, layer)
        K, V = t.kv_rows(reqs, [1] * len(reqs), layer)
        out = torch.full((len(reqs), t.Hq, t.d), float("nan"), dtype=torch.bfloat16, device="cuda")
        assert t.p.decode_append_attention(layer, reqs, bits_to_torch(K), bits_to_torch(V), bits_to_torch(q),
                                           out, t.scale) == 0
        staged.append((layer, q, K, V))
        outs.append(out)
    torch.cuda.synchronize()
    for (layer, q, K, V), out in zip(staged, outs):
        assert t.o.append(layer, reqs, [1] * len(reqs), K, V) == 0
        rc, ref = t.o.attention(layer, reqs, q, t.scale)
        assert rc == 0
        check_attention(torch_to_bits(out), ref, f"fused layer {layer}")


def _run_mixed(t, reqs):
    """fused(2), plain(2) [must not overlap], plain(1), fused(1)... on the pending +1 token of
    layers 2 and 1 (layers 0 and 3 appended up front without attention)."""
    import torch
    for layer in (0, 3):
        K, V = t.kv_rows(reqs, [1] * len(reqs), layer)
        assert t.o.append(layer, reqs, [1] * len(reqs), K, V) == 0
        assert t.p.append(layer, reqs, [1] * len(reqs), bits_to_torch(K), bits_to_torch(V)) == 0
    seq = [(2, True), (2, False), (0, False), (1, True), (3, False), (1, False), (0, False), (2, False)]
    staged, outs = [], []
    for layer, fused in seq:
        q = t.q_bits(reqs, layer)
        out = torch.full((len(reqs), t.Hq, t.d), float("nan"), dtype=torch.bfloat16, device="cuda")
        if fused:
            K, V = t.kv_rows(reqs, [1] * len(reqs), layer)
            rc = t.p.decode_append_attention(layer, reqs, bits_to_torch(K), bits_to_torch(V), bits_to_torch(q),
                                             out, t.scale)
        else:
            K = V = None
            rc = t.p.attention(layer, reqs, bits_to_torch(q), out, t.scale)
        assert rc == 0
        staged.append((layer, q, K, V))
        outs.append(out)
    torch.cuda.synchronize()
    for (layer, q, K, V), out in zip(staged, outs):
        if K is not None:
            assert t.o.append(layer, reqs, [1] * len(reqs), K, V) == 0
        rc, ref = t.o.attention(layer, reqs, q, t.scale)
        assert rc == 0
        check_attention(torch_to_bits(out), ref, f"mixed layer {layer}")

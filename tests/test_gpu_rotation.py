"""Rotated slabs (internal.h slab_slot): on the device, layer l of chunk c sits in
slab slot (l + floor(c/32)) mod L. Every kernel that touches KV bytes computes the slot, and the
host-visible images (read_chunk, host slots) stay canonical — so the oracle, which knows nothing
of the rotation, must still match bytes, tables and attention exactly / within R8 across
append, prefill, fused decode, deflate / inflate in both swap modes, migrate and release, on a
pool whose chunks span several rotation groups and an odd layer count."""
from __future__ import annotations

import numpy as np
import pytest

from tests.twin import Twin

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bulk", ["1", "0"], ids=["tma_migrate", "warp_migrate"])
@pytest.mark.parametrize("rotate", ["1", "0"])
def test_rotated_slabs_match_oracle(rotate, bulk, monkeypatch):
    monkeypatch.setenv("ELLM_ROTATE", rotate)
    monkeypatch.setenv("ELLM_D2D_BULK", bulk)  # migrate through the TMA bulk kernel or the warp kernel
    rng = np.random.default_rng(3)
    L, Hq, Hkv, d, T = 3, 8, 2, 128, 16          # chunk 48 KiB, slab 16 KiB
    R, MC, C, H = 6, 48, 224, 160                 # 7 rotation groups of 32 chunks
    t = Twin(L, Hq, Hkv, d, T, C, C, R, MC, H, seed=9, needle=False)
    lens = [300, 517, 410, 600, 333, 488]
    assert t.reserve(list(range(R)), lens) == 0
    t.append_all_layers(list(range(R)), lens)
    t.check_bytes()
    for l in range(L):
        t.attention(l, list(range(R)))
    # swap-out with the SM copy kernel, swap-in with the copy engines (and the reverse), and both
    # through the copy engines of the side context (swap mode 3)
    for out_mode, in_mode, r in ((0, 1, 2), (1, 0, 4), (3, 3, 5)):
        assert t.p.set_swap_mode(out_mode) == 0
        rc, slots = t.deflate(t.o.table(r)[0].tolist()[::-1])
        assert rc == 0
        t.check_bytes()
        assert t.p.set_swap_mode(in_mode) == 0
        assert t.inflate(slots[::2])[0] == 0
        assert t.inflate(slots[1::2])[0] == 0
        t.check_tables()
        t.check_bytes()
    # compaction: the highest USED chunks to the lowest FREE ids (crosses rotation groups)
    assert t.release(1) == 0
    used = sorted(c for r in range(R) for c in t.o.table(r)[0].tolist() if c >= 0)
    free = sorted(set(range(C)) - set(used))
    k = min(20, len(free))
    assert t.migrate(used[::-1][:k], free[:k]) == 0
    t.check_tables()
    t.check_bytes()
    # chunked prefill (tcgen05, multi-chunk TMA boxes) and fused decode over the moved chunks
    assert t.reserve([0, 3], [150, 90]) == 0
    t.append_all_layers([0, 3], [150, 90])
    for l in range(L):
        t.prefill(l, [0, 3], [150, 90], rng)
    live = [r for r in range(R) if t.lens[r] > 0]
    assert t.reserve(live, [1] * len(live)) == 0
    for l in range(L):
        t.decode_fused(l, live)
    t.check_bytes()

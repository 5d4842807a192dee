"""f1 — VMM-overhead hiding: speculative pre-mapping and
asynchronous unmapping move driver calls off pool_grow / pool_shrink without changing any result.
Ownership and tables are compared with the oracle after every op (the oracle has no notion of
mapping: pool_grow / pool_shrink are O9), bytes are read back through the tables (I4), and
attention is checked against the fp64 oracle on chunks whose memory was pre-mapped or taken
over from a unit awaiting its unmap (multi-mapping).

Geometry: L=2, Hq=8, Hkv=2, d=128, T=16 -> 32 KiB chunks; map unit = 2 MiB = 64 chunks."""
import numpy as np
import pytest

from tests.twin import Twin

pytestmark = pytest.mark.gpu

U = 2 << 20  # map unit bytes


def make(monkeypatch, delay_us, C=512, Ckv=128, R=4, MC=200, H=16, seed=3):
    # the worker-delay knob makes "right after the call" observations deterministic
    monkeypatch.setenv("ELLM_VMM_WORKER_DELAY_US", str(delay_us))
    return Twin(2, 8, 2, 128, 16, C, Ckv, R, MC, H, seed=seed, map_unit_bytes=U)


def test_premap_grow_makes_no_driver_call(monkeypatch):
    t = make(monkeypatch, 300_000)
    s = t.p.stats()
    assert s["mapped_bytes"] == 2 * U and s["n_map"] == 2 and s["premapped_bytes"] == 0
    assert t.p.set_vmm_overlap(U, False) == 0
    assert t.p.vmm_sync() == 0
    s = t.p.stats()
    assert s["premapped_bytes"] == U and s["mapped_bytes"] == 3 * U and s["n_map"] == 3
    assert t.grow(64) == 0                         # chunks 128..191 = the pre-mapped unit 2
    s = t.p.stats()
    assert s["n_map"] == 3 and s["premap_hits"] == 1 and s["premapped_bytes"] == 0
    assert t.p.vmm_sync() == 0                     # worker refills the window with unit 3
    s = t.p.stats()
    assert s["n_map"] == 4 and s["premapped_bytes"] == U and s["mapped_bytes"] == 4 * U
    assert t.reserve([0, 1], [16 * 150, 16 * 20]) == 0   # r0 reaches into the grown unit
    t.append_all_layers([0, 1], [16 * 150, 16 * 20])
    t.check_tables()
    t.check_bytes()
    t.attention(1, [0, 1])


def test_async_unmap_returns_before_unmapping(monkeypatch):
    t = make(monkeypatch, 300_000)
    assert t.p.set_vmm_overlap(0, True) == 0
    assert t.grow(128) == 0                        # units 2, 3 mapped on the caller's thread
    assert t.reserve([0], [16 * 40]) == 0
    t.append_all_layers([0], [16 * 40])
    s0 = t.p.stats()
    assert s0["mapped_bytes"] == 4 * U
    assert t.shrink(128) == 0                      # FREE 128..255 -> ACT: units 2, 3 all-ACT
    s = t.p.stats()
    assert s["mapped_bytes"] == 4 * U and s["pending_unmap"] == 2 and s["n_unmap"] == 0
    assert s["crit_vmm_ns"] == s0["crit_vmm_ns"]   # no unmap / device sync on the caller
    assert t.p.vmm_sync() == 0
    s = t.p.stats()
    assert s["mapped_bytes"] == 2 * U and s["pending_unmap"] == 0 and s["n_unmap"] == 2
    t.check_tables()
    t.check_bytes()
    t.attention(0, [0])


def test_grow_takes_handle_of_unit_awaiting_unmap(monkeypatch):
    t = make(monkeypatch, 300_000, C=320)
    assert t.grow(128) == 0                        # units 0..3 KV
    assert t.reserve([0, 1], [16 * 192, 16 * 64]) == 0   # r0 -> 0..191, r1 -> 192..255
    t.append_all_layers([0, 1], [16 * 192, 16 * 64])
    assert t.release(0) == 0
    assert t.p.set_vmm_overlap(0, True) == 0
    assert t.shrink(64) == 0                       # 128..191 -> ACT: unit 2 pending
    assert t.p.vmm_sync() == 0 and t.p.stats()["mapped_bytes"] == 3 * U
    t.release(1)
    assert t.shrink(64) == 0                       # 192..255 -> ACT: unit 3 pending (worker delayed)
    assert t.p.stats()["pending_unmap"] == 1
    assert t.grow(64) == 0                         # 128..191: unit 2 backed by unit 3's handle
    s = t.p.stats()
    assert s["n_steal"] == 1 and s["mapped_bytes"] == 4 * U and s["pending_unmap"] == 1
    assert t.reserve([2], [16 * 150]) == 0         # 0..149: reaches into unit 2
    t.append_all_layers([2], [16 * 150])
    t.check_tables()
    t.check_bytes()
    t.attention(0, [2])
    assert t.p.vmm_sync() == 0                     # unit 3's VA unmapped, handle kept by unit 2
    s = t.p.stats()
    assert s["mapped_bytes"] == 3 * U and s["pending_unmap"] == 0
    t.check_bytes()
    t.attention(1, [2])


def test_random_elastic_ops_with_overlap(monkeypatch):
    """test_elastic_ops_bytes_and_attention's op mix with pre-mapping + async unmap on and no
    worker delay: the worker races the caller; every result must still match the oracle."""
    rng = np.random.default_rng(11)
    R, C = 6, 512
    t = make(monkeypatch, 0, C=C, Ckv=128, R=R, MC=120, H=32, seed=9)
    assert t.p.set_vmm_overlap(U, True) == 0
    for it in range(80):
        op = int(rng.integers(0, 8))
        if op <= 1:
            reqs = [int(x) for x in rng.choice(R, size=int(rng.integers(1, 3)), replace=False)]
            nn = [int(x) for x in rng.integers(16, 16 * 40, size=len(reqs))]
            if t.reserve(reqs, nn) == 0:
                t.append_all_layers(reqs, nn)
        elif op == 2:
            used = [c for r in range(R) for c in t.o.table(r)[0].tolist() if c >= 0]
            if used:
                t.deflate(rng.choice(used, size=min(len(used), int(rng.integers(1, 6))), replace=False))
        elif op == 3:
            hs = [-e - 2 for r in range(R) for e in t.o.table(r)[0].tolist() if e <= -2]
            if hs:
                t.inflate(rng.choice(hs, size=min(len(hs), int(rng.integers(1, 6))), replace=False))
        elif op == 4:
            t.release(int(rng.integers(0, R)))
        elif op == 5:
            t.grow(int(rng.integers(1, 160)))
        else:
            t.shrink(int(rng.integers(1, 160)))
        if it % 8 == 7:
            t.check_tables()
            t.check_bytes()
    assert t.p.vmm_sync() == 0
    t.check_tables()
    t.check_bytes()
    live = [r for r in range(R) if t.o.table(r)[1] > 0 and all(e >= 0 for e in t.o.table(r)[0].tolist())]
    if live:
        t.attention(1, live)
    s = t.p.stats()
    assert s["premapped_bytes"] <= U and s["pending_unmap"] == 0

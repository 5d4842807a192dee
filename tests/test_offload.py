"""Layer-wise pipelined offload: offload_begin / offload_layer x L /
offload_commit must reach exactly the state of ellm_deflate on the same chunk list (tables,
stats, host-slot bytes) — the oracle's deflate (O5) is the reference."""
import numpy as np
import pytest

import oracle
from oracle import Oracle
from paper_2506_15155_b200 import ellm


def test_offload_metadata_matches_oracle_deflate():
    L = 3
    o = Oracle(L, 4, 2, 64, 16, 40, 40, 3, 12, 24)
    p = ellm.Pool(ellm.DEVICE_NONE, L, 4, 2, 64, 16, 40, 40, 3, 12, 24)
    for x in (o, p):
        assert x.reserve([0, 1, 2], [70, 40, 100]) == 0
    ids = p.table(2)[0].tolist()[::-1]
    rc_o, slots_o = o.deflate(ids)
    rc, slots = p.offload_begin(ids)
    assert rc == rc_o == 0 and slots.tolist() == slots_o.tolist()
    assert p.offload_begin(ids[:1])[0] == ellm.ALREADY_MAPPED     # already being offloaded
    assert p.deflate(ids[:1])[0] == ellm.IN_USE
    assert p.offload_commit(ids) == ellm.INVALID_ARG             # layers not copied yet
    for l in range(L):
        assert p.offload_layer(l, ids) == 0
    assert p.offload_layer(L, ids) == ellm.OUT_OF_RANGE
    assert p.offload_layer(0, [p.table(0)[0][0]]) == ellm.NOT_MAPPED
    assert p.offload_commit(ids) == 0
    for r in range(3):
        assert p.table(r)[0].tolist() == o.table(r)[0].tolist()
    so, sp = o.stats(), p.stats()
    assert all(so[k] == sp[k] for k in so)
    # release of a request with an offload in progress returns its reserved slots
    rc, sl = p.offload_begin(p.table(0)[0].tolist())
    assert rc == 0 and p.stats()["host_used"] == len(ids) + len(sl)
    assert p.release(0) == 0 and p.stats()["host_used"] == len(ids)


def test_offload_commit_needs_every_layer_not_a_count():
    """offload_commit checks which layers were copied (a per-chunk bitset), not how many calls
    were made: copying layer 0 L times does not make layers 1..L-1 copied."""
    L = 3
    p = ellm.Pool(ellm.DEVICE_NONE, L, 4, 2, 64, 16, 40, 40, 3, 12, 24)
    assert p.reserve([0], [70]) == 0
    ids = p.table(0)[0].tolist()
    assert p.offload_begin(ids)[0] == 0
    for _ in range(L):
        assert p.offload_layer(0, ids) == 0
    assert p.offload_commit(ids) == ellm.INVALID_ARG
    assert p.offload_layer(2, ids) == 0
    assert p.offload_commit(ids) == ellm.INVALID_ARG      # layer 1 still missing
    assert p.offload_layer(1, ids[1:]) == 0               # ... for one chunk
    assert p.offload_commit(ids) == ellm.INVALID_ARG
    assert p.offload_layer(1, ids[:1]) == 0
    assert p.offload_commit(ids) == 0
    # a fresh offload of other chunks starts with no layer marked
    assert p.reserve([1], [40]) == 0
    ids1 = p.table(1)[0].tolist()
    assert p.offload_begin(ids1)[0] == 0
    assert p.offload_layer(0, ids1) == 0 and p.offload_layer(1, ids1) == 0
    assert p.offload_commit(ids1) == ellm.INVALID_ARG


@pytest.mark.gpu
@pytest.mark.parametrize("mode,rotate", [(0, "0"), (1, "0"), (0, "1"), (1, "1"), (3, "1")])
def test_offload_layerwise_bytes_overlapped_with_appends(mode, rotate, monkeypatch):
    """Prefill request 1 layer by layer on the compute stream while each finished layer is
    offloaded on a second stream (event per layer); after commit the host slots hold exactly
    what the oracle's deflate holds. SM copy kernel (mode 0) or copy engines (mode 1; mode 3 adds
    the fetch-back through the side context), canonical or rotated slabs (request 1's chunks sit
    in the second rotation group)."""
    import torch
    from inputs import gen
    from tests.twin import Twin, bits_to_torch
    monkeypatch.setenv("ELLM_ROTATE", rotate)
    L, Hq, Hkv, d, T = 4, 32, 8, 128, 16
    t = Twin(L, Hq, Hkv, d, T, 64, 64, 2, 40, 32, seed=17)
    assert t.p.set_swap_mode(mode) == 0
    assert t.reserve([0, 1], [600, 300]) == 0
    t.append_all_layers([0], [600])
    ids = t.p.table(1)[0].tolist()
    rc, slots = t.p.offload_begin(ids)
    assert rc == 0
    s_off = torch.cuda.Stream()
    for l in range(L):  # oracle append + product append on the compute stream, offload on s_off
        K, V = t.kv_rows([1], [300], l)
        assert t.o.append(l, [1], [300], K, V) == 0
        assert t.p.append(l, [1], [300], bits_to_torch(K), bits_to_torch(V)) == 0
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        s_off.wait_event(ev)
        assert t.p.offload_layer(l, ids, s_off) == 0
    assert t.p.offload_commit(ids, s_off) == 0
    rc_o, slots_o = t.o.deflate(ids)
    assert rc_o == 0 and slots_o.tolist() == slots.tolist()
    torch.cuda.synchronize()
    t.check_tables()
    t.check_bytes()
    assert t.attention(0, [1])[0] == -5        # now host-resident
    rc, back = t.inflate(slots)
    assert rc == 0
    t.check_bytes()
    t.attention(L - 1, [0, 1])

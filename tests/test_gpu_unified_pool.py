"""f3 — unified pool with activation eTensors.

Activation slots are runs of ACT chunks of the same pool the KV cache lives in; ownership and
tables are compared with the oracle (O9-O11) after every op, KV bytes are read back through the
tables (I4) and attention is checked against the fp64 oracle on chunks that held activations
just before. Inflation from ended activation slots must make no driver call: the memory is
already mapped, only the owner label changes (the paper's zero-overhead ownership transfer).

Geometry: L=2, Hq=8, Hkv=2, d=128, T=16 -> 32 KiB chunks; map unit = 2 MiB = 64 chunks."""
import numpy as np
import pytest

from tests.twin import Twin

pytestmark = pytest.mark.gpu

U = 2 << 20


def test_activation_slots_then_zero_overhead_inflation():
    t = Twin(2, 8, 2, 128, 16, 512, 128, 4, 200, 8, seed=4, map_unit_bytes=U)
    cb = t.p.chunk_bytes
    s0 = t.p.stats()
    assert s0["n_map"] == 2                          # units 0, 1 (KV chunks 0..127)
    assert t.act_alloc(100) == (0, 412)              # top of the pool: 412..511 (units 6, 7)
    assert t.p._last_act_ptr == t.p.base() + 412 * cb
    s = t.p.stats()
    assert s["n_map"] == 4 and s["act_used"] == 100
    states = t.p.chunk_states()
    assert states[412:].tolist() == [3] * 100 and states[128:412].tolist() == [2] * 284
    assert t.grow(300) == -3                         # only 284 idle ACT chunks (128..411)
    assert t.grow(284) == 0                          # units 2..5 fresh, unit 6 already mapped
    assert t.p.stats()["n_map"] == 8
    assert t.act_free(412) == 0
    s = t.p.stats()
    assert s["act_used"] == 0 and s["act_cached_bytes"] == U   # unit 7 (unit 6 also holds KV)
    assert t.grow(100) == 0                          # 412..511: the ended slot's chunks
    s = t.p.stats()
    assert s["n_map"] == 8 and s["act_cached_bytes"] == 0      # no driver call
    # KV into the reclaimed chunks: r0 takes 0..199, r1 200..399, r2 400..511
    lens = [200 * 16, 200 * 16, 100 * 16 + 5]
    assert t.reserve([0, 1, 2], lens) == 0
    assert t.o.table(2)[0].tolist()[-1] == 500
    t.append_all_layers([0, 1, 2], lens)
    t.check_tables()
    t.check_bytes()
    t.attention(1, [0, 1, 2])


def test_shrink_then_activation_slot_then_trim():
    t = Twin(2, 8, 2, 128, 16, 256, 256, 2, 100, 0, seed=6, map_unit_bytes=U)
    assert t.reserve([0], [70 * 16]) == 0            # 0..69
    t.append_all_layers([0], [70 * 16])
    assert t.shrink(186) == 0                        # 70..255 -> ACT; units 2, 3 unmapped now
    s = t.p.stats()
    assert s["n_unmap"] == 2 and s["mapped_bytes"] == 2 * U
    assert t.act_alloc(40) == (0, 216)               # 216..255: unit 3 mapped again
    assert t.act_alloc(100) == (0, 116)              # 116..215: units 1..3
    assert t.p.stats()["mapped_bytes"] == 4 * U
    assert t.act_free(216) == 0 and t.act_free(116) == 0
    assert t.p.stats()["act_cached_bytes"] == 2 * U  # units 2, 3 (unit 1 holds KV)
    assert t.p.act_trim() == 0
    s = t.p.stats()
    assert s["act_cached_bytes"] == 0 and s["mapped_bytes"] == 2 * U
    t.check_tables()
    t.check_bytes()
    t.attention(0, [0])


def test_torch_mempool_tensors_live_in_activation_slots():
    """torch's caching allocator on top (activation pool keeps BFC): a MemPool built on
    the pool's pluggable-allocator hooks places tensors in activation slots of the pool VA;
    they compute correctly; when torch releases its segments the chunks are idle ACT again and
    inflation takes them without a driver call."""
    import torch
    from paper_2506_15155_b200 import ellm
    C = 2048                                         # 2048 x 32 KiB = 64 MiB (32 units)
    p = ellm.Pool(0, 2, 8, 2, 128, 16, C, 256, 2, 100, 0, U)
    lo, hi = p.base(), p.base() + C * p.chunk_bytes
    mp = p.activation_mempool()
    g = torch.Generator(device="cpu").manual_seed(0)
    a_cpu = torch.randn(1024, 1024, generator=g)
    w = torch.ones(8, 8, device="cuda")
    w = w @ w                                        # cuBLAS workspace outside the MemPool
    with torch.cuda.use_mem_pool(mp):
        a = a_cpu.cuda()
        b = a @ a                                    # 4 MiB operands / result
        c = torch.empty(1000, device="cuda")
        c.fill_(3.0)
    assert all(lo <= t_.data_ptr() < hi for t_ in (a, b, c))
    torch.cuda.synchronize()
    s = p.stats()
    assert s["act_used"] > 0 and s["act"] == C - 256
    ref = a_cpu.double() @ a_cpu.double()
    assert torch.allclose(b.cpu().double(), ref, atol=1e-2, rtol=1e-3)
    assert float(c.sum()) == 3000.0
    used = s["act_used"]
    assert p.grow(C - 256 - used + 1) == ellm.NO_CHUNKS   # live activation chunks are not reclaimable
    del a, b, c                                      # no outstanding allocations: the MemPool's
    del mp                                           # segments go back through ellm_torch_free
    torch._C._cuda_clearCublasWorkspaces()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    s = p.stats()
    assert s["act_used"] == 0
    n_map = s["n_map"]
    assert p.grow(C - 256) == ellm.OK                # all of it, including the ex-activation units
    s = p.stats()
    cached_units = used // 64                        # whole units activations had mapped
    assert s["n_map"] - n_map <= (C - 256) // 64 - cached_units + 1
    ellm.ellm_torch_set_pool(None)
    p.close()

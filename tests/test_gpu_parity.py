"""GPU parity: the CUDA path (through the C ABI) against the oracle on identical seeded
inputs. Integer / byte state bit-exact; attention within the BASELINE.json tolerance."""
import ctypes

import numpy as np
import pytest

from inputs import gen
from tests.twin import Twin, bits_to_torch, torch_to_bits, check_attention

pytestmark = pytest.mark.gpu


def test_device_generator_matches_numpy_bit_exactly():
    import torch
    from inputs import workload
    lib = workload.gen_lib()
    for (seed, r, p0, n, l, kv, h0, nh, d, group, nr) in [
            (1, 3, 0, 300, 2, 0, 0, 8, 128, 4, 300), (1, 3, 0, 300, 2, 1, 0, 8, 128, 4, 300),
            (5, 17, 1000, 77, 31, 0, 4, 2, 128, 8, 2000), (0, 0, 5, 40, 0, 1, 1, 1, 64, 2, 45)]:
        out = torch.empty((n, nh, d), dtype=torch.bfloat16, device="cuda")
        assert lib.ellm_gen_kv(seed, r, p0, n, l, kv, h0, nh, d, group, nr, out.data_ptr(), 0) == 0
        want = gen.kv_bits(seed, r, np.arange(p0, p0 + n), l, kv, range(h0, h0 + nh), d, group, nr)
        assert np.array_equal(torch_to_bits(out), want)
    q = torch.empty((6, 128), dtype=torch.bfloat16, device="cuda")
    assert lib.ellm_gen_q(9, 4, 3, 10, 6, 128, q.data_ptr(), 0) == 0
    assert np.array_equal(torch_to_bits(q), gen.q_bits(9, 4, 3, range(10, 16), 128))


def test_c1_flow():
    """BASELINE.json configs[0]: prefill 4 requests {17,64,129,300}, 3 decode steps,
    deflate 8 chunks of r3, NOT_RESIDENT, inflate, attention."""
    t = Twin(1, 4, 2, 64, 16, 64, 64, 4, 32, 64, seed=0)
    lens = [17, 64, 129, 300]
    assert t.reserve([0, 1, 2, 3], lens) == 0
    t.append_all_layers([0, 1, 2, 3], lens)
    t.check_tables()
    t.check_bytes()
    t.attention(0, [0, 1, 2, 3])
    for _ in range(3):
        assert t.reserve([0, 1, 2, 3], [1, 1, 1, 1]) == 0
        t.append_all_layers([0, 1, 2, 3], [1, 1, 1, 1])
        t.attention(0, [0, 1, 2, 3])
    t.check_tables()
    ids = t.o.table(3)[0][:8].tolist()
    assert ids == list(range(15, 23))
    rc, slots = t.deflate(ids)
    assert rc == 0 and slots.tolist() == list(range(8))
    t.check_bytes()
    assert t.attention(0, [3])[0] == -5
    t.attention(0, [0, 1, 2])
    rc, back = t.inflate(slots)
    assert rc == 0 and back.tolist() == ids
    t.check_tables()
    t.check_bytes()
    t.attention(0, [3, 2, 1, 0])


SHAPES = [  # (L, Hq, Hkv, d, T)
    (2, 32, 8, 128, 16),    # LLaMA-3-8B geometry (HB 8, TT 16)
    (2, 64, 8, 128, 32),    # 70B geometry, group 8
    (1, 16, 4, 128, 32),    # 8B at 2-way shard (HB 4, TT 32)
    (1, 8, 2, 128, 16),     # 4-way shard, multi-piece stages (T < TT)
    (1, 8, 1, 128, 256),    # 70B at 8-way shard (HB 1, TT 128)
    (1, 4, 1, 128, 16),     # HB 1 with 8 pieces per stage
    (2, 4, 2, 64, 16),      # C1 geometry
    (1, 64, 8, 64, 16),     # d 64, group 8
    (1, 8, 4, 64, 64),
    (1, 16, 16, 128, 16),   # MHA, 2 head groups (HG 2)
]


@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_shapes_ragged(shape):
    L, Hq, Hkv, d, T = shape
    lens = [1, 15, 16, 17, 127, 300, 1001, 2049]
    R = len(lens)
    mc = max((x + 40 + T - 1) // T for x in lens)
    C = R * mc + 4
    t = Twin(L, Hq, Hkv, d, T, C, C, R, mc, 8, seed=11)
    reqs = list(range(R))
    assert t.reserve(reqs, lens) == 0
    t.append_all_layers(reqs, lens)
    t.check_tables()
    t.check_bytes()
    for l in range(L):
        t.attention(l, reqs)
    # two decode steps and a permuted / duplicated request list
    for _ in range(2):
        assert t.reserve(reqs, [1] * R) == 0
        t.append_all_layers(reqs, [1] * R)
    t.attention(L - 1, [7, 3, 3, 0, 5])
    t.check_bytes()


def test_long_single_request_spans_all_ctas():
    t = Twin(1, 32, 8, 128, 16, 1300, 1300, 2, 1300, 0, seed=3)
    assert t.reserve([0], [20000]) == 0
    t.append_all_layers([0], [20000])
    t.attention(0, [0])
    assert t.reserve([1], [5]) == 0
    t.append_all_layers([1], [5])
    t.attention(0, [1, 0, 1])


def test_elastic_ops_bytes_and_attention():
    """Random deflate / inflate / migrate / release / grow / shrink with byte-exact checks
    after each op and attention after the sequence."""
    rng = np.random.default_rng(7)
    L, Hq, Hkv, d, T = 2, 8, 2, 128, 16
    R, MC, C, H = 6, 12, 64, 24
    t = Twin(L, Hq, Hkv, d, T, C, 48, R, MC, H, seed=5)
    for it in range(60):
        op = int(rng.integers(0, 7))
        if op <= 1:
            reqs = [int(x) for x in rng.choice(R, size=int(rng.integers(1, 3)), replace=False)]
            nn = [int(x) for x in rng.integers(1, 40, size=len(reqs))]
            if t.reserve(reqs, nn) == 0:
                t.append_all_layers(reqs, nn)
        elif op == 2:
            used = [c for r in range(R) for c in t.o.table(r)[0].tolist() if c >= 0]
            if used:
                t.deflate(rng.choice(used, size=min(len(used), int(rng.integers(1, 4))), replace=False))
        elif op == 3:
            hs = [-e - 2 for r in range(R) for e in t.o.table(r)[0].tolist() if e <= -2]
            if hs:
                t.inflate(rng.choice(hs, size=min(len(hs), int(rng.integers(1, 4))), replace=False))
        elif op == 4:
            used = sorted(c for r in range(R) for c in t.o.table(r)[0].tolist() if c >= 0)
            if used:
                # compaction step: highest USED -> lowest id not in use (may be ACT: NOT_MAPPED)
                dst = min(set(range(C)) - set(used))
                t.migrate([used[-1]], [dst])
        elif op == 5:
            t.release(int(rng.integers(0, R)))
        else:
            t.grow(int(rng.integers(0, 3))) if rng.integers(0, 2) else t.shrink(int(rng.integers(0, 3)))
        t.check_tables()
        if it % 6 == 0:
            t.check_bytes()
    t.check_bytes()
    resident = [r for r in range(R) if t.lens[r] > 0 and all(e >= 0 for e in t.o.table(r)[0])]
    for l in range(L):
        if resident:
            t.attention(l, resident)


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_swap_modes_roundtrip(mode):
    t = Twin(2, 32, 8, 128, 16, 40, 40, 3, 12, 40, seed=2)
    assert t.p.set_swap_mode(mode) == 0, t.p.last_cuda_error()
    assert t.reserve([0, 1, 2], [100, 60, 150]) == 0
    t.append_all_layers([0, 1, 2], [100, 60, 150])
    before = t.attention(1, [0, 1, 2])[1][0]
    ids = t.o.table(2)[0].tolist()
    rc, slots = t.deflate(ids[::-1])
    assert rc == 0
    t.check_bytes()
    rc, back = t.inflate(slots[::2])
    rc, back2 = t.inflate(slots[1::2])
    t.check_tables()
    t.check_bytes()
    after = t.attention(1, [0, 1, 2])[1][0]
    assert np.array_equal(before[:2], after[:2])


def test_vmm_grow_shrink_and_alias_view():
    """pool_grow / pool_shrink map and unmap 2 MiB chunks (cuMemMap/cuMemUnmap); the alias
    view maps a request's chunks contiguously (the paper's KV eTensor)."""
    import torch
    t = Twin(32, 32, 8, 128, 16, 16, 6, 2, 8, 2, seed=4, map_unit_bytes=2 << 20)
    assert t.p.chunk_bytes == 2 << 20
    s0 = t.p.stats()
    assert s0["mapped_bytes"] == 6 * (2 << 20) and s0["n_map"] == 6
    assert t.reserve([0], [100]) == -3          # 7 chunks > 6 FREE: NO_CHUNKS
    assert t.grow(4) == 0
    assert t.p.stats()["mapped_bytes"] == 10 * (2 << 20)
    assert t.reserve([0], [100]) == 0
    t.append_all_layers([0], [100])
    t.check_bytes()
    rc, ptr = t.p.alias_request(0)
    assert rc == 0 and ptr
    nbytes = 7 * t.p.chunk_bytes

    class _View:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}

    contig = torch.as_tensor(_View(), device="cuda").cpu().numpy()
    tab = t.o.table(0)[0]
    for i, c in enumerate(tab.tolist()):
        assert np.array_equal(contig[i * t.p.chunk_bytes:(i + 1) * t.p.chunk_bytes], t.p.read_chunk(c))
    assert t.p.unalias_request(0) == 0
    assert t.shrink(3) == 0
    s1 = t.p.stats()
    assert s1["n_unmap"] == 3 and s1["act"] == 9
    assert t.shrink(1) == -8
    t.check_bytes()
    t.attention(5, [0])


def test_error_codes_match_oracle_on_device():
    t = Twin(1, 4, 2, 64, 16, 16, 16, 3, 8, 2, seed=1)
    assert t.reserve([0, 1], [40, 20]) == 0
    t.append_all_layers([0, 1], [40, 20])
    assert t.reserve([3], [1]) == -2
    assert t.reserve([0, 0], [1, 1]) == -1
    assert t.reserve([0], [200]) == -2
    assert t.reserve([2, 1], [128, 70]) == -3   # 8 + 4 new chunks > 11 FREE
    assert t.append(0, [0], [3]) == -1
    assert t.attention(0, [2])[0] == -1
    assert t.deflate([15])[0] == -6
    assert t.deflate([0, 1, 2])[0] == -4
    assert t.migrate([0], [1]) == -7
    assert t.inflate([1])[0] == -6
    t.check_tables()
    t.check_bytes()


FUSED_SHAPES = [(2, 32, 8, 128, 16), (1, 64, 8, 128, 32), (1, 8, 2, 128, 16), (1, 8, 1, 128, 256),
                (2, 4, 2, 64, 16), (1, 16, 16, 128, 16)]


@pytest.mark.parametrize("shape", FUSED_SHAPES, ids=[str(s) for s in FUSED_SHAPES])
def test_fused_decode_append_attention(shape):
    """ellm_decode_append_attention == kv_append + attention: bytes bit-exact (the new row lands
    in its chunk), attention within tolerance, for decode steps crossing chunk boundaries."""
    L, Hq, Hkv, d, T = shape
    lens = [1, 15, 16, 31, 300, 2047]
    R = len(lens)
    mc = max((x + 40 + T - 1) // T for x in lens)
    t = Twin(L, Hq, Hkv, d, T, R * mc + 4, R * mc + 4, R, mc, 0, seed=21)
    reqs = list(range(R))
    assert t.reserve(reqs, lens) == 0
    t.append_all_layers(reqs, lens)
    for step in range(20):
        assert t.reserve(reqs, [1] * R) == 0
        for l in range(L):
            assert t.decode_fused(l, reqs[::-1] if step % 2 else reqs) == 0
    t.check_tables()
    t.check_bytes()
    # precondition: the latest reservation must be exactly one token
    assert t.reserve([0], [2]) == 0
    assert t.decode_fused(0, [0]) == -1


@pytest.mark.parametrize("div", [8, 3])
def test_dynamic_tail_schedule(div, monkeypatch):
    """The optional dynamic-tail schedule (ELLM_ATTN_DYN_DIV): the last
    tiles/div tiles of every request are claimed in units by whichever CTA is free; results
    must match the oracle exactly as the static schedule does (also fused decode)."""
    monkeypatch.setenv("ELLM_ATTN_DYN_DIV", str(div))
    # short requests between long ones have no dynamic tiles: units span over them
    lens = [4000, 3001, 17, 2500, 1, 40, 1800, 16, 33, 3000, 5, 2222]
    R = len(lens)
    t = Twin(1, 32, 8, 128, 16, 1400, 1400, R, 260, 0, seed=13)
    reqs = list(range(R))
    assert t.reserve(reqs, lens) == 0
    t.append_all_layers(reqs, lens)
    for _ in range(6):
        t.attention(0, reqs)           # ticket counter advances across launches
    assert t.reserve(reqs, [1] * R) == 0
    assert t.decode_fused(0, reqs[::-1]) == 0
    t.check_bytes()


def test_map_units_follow_ownership():
    """Default map units (64 MiB = 32 chunks of 2 MiB): a unit is mapped when its first chunk
    becomes KV and unmapped when its last chunk returns to ACT; bytes survive."""
    MB2 = 2 << 20
    t = Twin(32, 32, 8, 128, 16, 100, 40, 3, 16, 0, seed=8)
    s = t.p.stats()
    assert s["mapped_bytes"] == 2 * 32 * MB2 and s["n_map"] == 2      # chunks 0..63 -> units 0, 1
    assert t.grow(30) == 0                                             # chunks 40..69 -> unit 2
    assert t.p.stats()["n_map"] == 3
    assert t.reserve([0, 1], [16 * 16, 16 * 10]) == 0
    t.append_all_layers([0, 1], [16 * 16, 16 * 10])
    assert t.shrink(44) == 0                                           # FREE 26..69 -> ACT
    s = t.p.stats()
    assert s["n_unmap"] == 2 and s["mapped_bytes"] == 32 * MB2        # units 1, 2 released
    assert t.grow(40) == 0                                             # 26..65: units 1, 2 back
    assert t.p.stats()["n_map"] == 5
    t.check_tables()
    t.check_bytes()
    t.attention(31, [0, 1])


@pytest.mark.parametrize("dyn", ["0", "16"])
def test_attention_is_deterministic(dyn, monkeypatch):
    """DESIGN.md R17: a launch's output bits do not depend on which CTA claimed which work (the
    merge order is fixed by record id) — repeated launches, with and without dynamic tickets,
    give identical bits, and they are within R8 of the oracle."""
    import torch
    monkeypatch.setenv("ELLM_ATTN_DYN_DIV", dyn)
    t = Twin(1, 32, 8, 128, 16, 1100, 1100, 4, 400, 0, seed=13)
    lens = [6000, 77, 2900, 1234]  # 640 tiles >= 4 x #SM: the dynamic tail engages with dyn=16
    assert t.reserve([0, 1, 2, 3], lens) == 0
    t.append_all_layers([0, 1, 2, 3], lens)
    rc, (first, _) = t.attention(0, [2, 0, 3, 1])
    assert rc == 0
    q = bits_to_torch(t.q_bits([2, 0, 3, 1], 0))
    for _ in range(4):
        out = torch.empty((4, 32, 128), dtype=torch.bfloat16, device="cuda")
        assert t.p.attention(0, [2, 0, 3, 1], q, out, t.scale) == 0
        torch.cuda.synchronize()
        assert np.array_equal(torch_to_bits(out), first)


def test_attention_list_longer_than_max_requests():
    """a request list with repeated ids may be longer than max_requests; the split-K
    state grows (device-synchronising) instead of being overrun, and every entry is correct."""
    t = Twin(1, 32, 8, 128, 16, 300, 300, 2, 150, 0, seed=19)
    assert t.reserve([0, 1], [1500, 333]) == 0
    t.append_all_layers([0, 1], [1500, 333])
    t.attention(0, [0, 1] * 5)           # 10 entries, max_requests 2
    t.attention(0, [1, 1, 1, 0] * 8)     # 32 entries: grows again
    t.attention(0, [1, 0])               # and the small list still works afterwards


@pytest.mark.parametrize("rotate", ["0", "1"])
def test_copy_engine_runs_match_oracle(rotate, monkeypatch):
    """The copy-engine swap path (pool.cpp issue_copies) merges a chunk list into one
    cudaMemcpyAsync per contiguous run and one cudaMemcpy2DAsync per evenly strided run. Lists
    mixing a consecutive run, a reversed run, strided ids and singletons — deflated into slots
    that are consecutive, then inflated from slots in a shuffled order (strided / scattered
    destinations) — must leave tables and bytes bit-exact with the oracle, canonical and with
    rotated slabs (per-chunk pieces listed piece-major)."""
    monkeypatch.setenv("ELLM_ROTATE", rotate)
    rng = np.random.default_rng(23)
    t = Twin(3, 8, 2, 128, 16, 160, 160, 4, 60, 160, seed=29)   # 48 KiB chunks, 16 KiB slabs
    t.p.set_swap_mode(1)
    lens = [900, 300, 700, 555]
    assert t.reserve(list(range(4)), lens) == 0
    t.append_all_layers(list(range(4)), lens)
    ids0 = t.o.table(0)[0].tolist()          # consecutive ids
    ids2 = t.o.table(2)[0].tolist()
    mixed = ids0[:10] + ids2[::-1][:8] + ids0[10:30:3] + [ids2[0]]
    rc, slots = t.deflate(mixed)
    assert rc == 0
    t.check_tables()
    t.check_bytes()
    order = rng.permutation(len(slots))
    rc, _ = t.inflate([int(slots[i]) for i in order[: len(order) // 2]])
    assert rc == 0
    rc, _ = t.inflate([int(slots[i]) for i in order[len(order) // 2:]][::-1])
    assert rc == 0
    t.check_tables()
    t.check_bytes()
    for l in range(3):
        t.attention(l, [0, 1, 2, 3])


def test_trace_and_split_weights_keep_results():
    """The timeline instrumentation (ellm_set_attn_trace) does not change a launch's bits; the
    split-weight knob (ellm_debug_attn_weights) changes the partition but stays within R8."""
    import torch
    t = Twin(1, 32, 8, 128, 16, 1100, 1100, 4, 400, 0, seed=31)
    lens = [6000, 300, 2900, 1234]
    assert t.reserve([0, 1, 2, 3], lens) == 0
    t.append_all_layers([0, 1, 2, 3], lens)
    rc, (plain, _) = t.attention(0, [0, 1, 2, 3])
    assert rc == 0
    G = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros((2, G, 8), dtype=torch.int64, device="cuda")
    assert t.p.set_attn_trace(buf, 2) == 0
    rc, (traced, _) = t.attention(0, [0, 1, 2, 3])
    assert rc == 0 and np.array_equal(traced, plain)
    stamps = buf[0].cpu().numpy()
    live = stamps[:, 0] > 0
    assert live.sum() > 0 and np.all(stamps[live, 5] >= stamps[live, 0])
    assert t.p.set_attn_trace(None, 0) == 0
    w = np.random.default_rng(3).uniform(0.5, 2.0, G)
    assert t.p.debug_attn_weights(w) == 0
    t.attention(0, [0, 1, 2, 3])             # checked against the oracle inside
    assert t.p.debug_attn_weights([]) == 0
    rc, (again, _) = t.attention(0, [0, 1, 2, 3])
    assert rc == 0 and np.array_equal(again, plain)

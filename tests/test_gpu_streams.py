"""Stream-ordered reuse (include/ellm.h "Conventions"): chunks freed by a deflate on one stream
and immediately handed to a reserve + append on another stream must not be overwritten
before the copy-out has read them; host slots freed by an inflate likewise."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _fill(pool, wl, r, n, stream):
    import torch
    from inputs import workload as W
    row = wl.hkv_local * wl.head_dim * 2
    kb = torch.empty((n, wl.hkv_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    vb = torch.empty_like(kb)
    s = stream.cuda_stream
    for l in range(wl.n_layers):
        W.gen_kv_device(wl, r, 0, n, l, 0, kb.data_ptr(), s)
        W.gen_kv_device(wl, r, 0, n, l, 1, vb.data_ptr(), s)
        assert pool.append(l, [r], [n], kb, vb, s) == 0
    del row
    return kb, vb


def _check_chunk(img, wl, r, i, T=16):
    from inputs import gen
    img = img.view(np.uint16).reshape(wl.n_layers, 2, wl.hkv_local, T, wl.head_dim)
    pos = np.arange(i * T, (i + 1) * T)
    for l in (0, wl.n_layers - 1):
        for kv in (0, 1):
            want = gen.kv_bits(wl.seed, r, pos, l, kv, range(wl.hkv_local), wl.head_dim, wl.group, 0)
            assert np.array_equal(img[l, kv].transpose(1, 0, 2), want), (r, i, l, kv)


@pytest.mark.parametrize("mode", [0, 3])
def test_deflate_then_reuse_on_another_stream(mode):
    """mode 0: SM copy kernels; mode 3: copy engines of the pool's side context (the copies run
    on another context's stream, ordered by events)."""
    import torch
    from inputs import workload as W
    from paper_2506_15155_b200 import ellm
    wl = W.Workload("streams", 32, 32, 8, 128, 2, 32000, seed=9, needle=False)
    n_chunks = 2000
    pool = ellm.Pool(0, 32, 32, 8, 128, 16, 2 * n_chunks + 8, 2 * n_chunks + 8, 2, n_chunks, n_chunks)
    assert pool.set_swap_mode(mode) == 0, pool.last_cuda_error()
    s0, s1, s2 = torch.cuda.current_stream(), torch.cuda.Stream(), torch.cuda.Stream()
    assert pool.reserve([0], [wl.context], s0.cuda_stream) == 0
    _fill(pool, wl, 0, wl.context, s0)
    torch.cuda.synchronize()
    ids_a = pool.table(0)[0].tolist()
    # ~4 GiB copy-out on s1, and request 1 immediately takes the freed chunks on s2
    rc, slots = pool.deflate(ids_a, s1.cuda_stream)
    assert rc == 0
    assert pool.reserve([1], [wl.context], s2.cuda_stream) == 0
    assert sorted(pool.table(1)[0].tolist()) == sorted(ids_a)[: len(ids_a)]  # lowest ids reused
    kb, vb = _fill(pool, wl, 1, wl.context, s2)
    torch.cuda.synchronize()
    for i in (0, 999, n_chunks - 1):
        _check_chunk(pool.read_host_slot(int(slots[i])), wl, 0, i)             # A intact on host
        _check_chunk(pool.read_chunk(int(pool.table(1)[0][i])), wl, 1, i)      # B in the chunks
    # inflate A back on s1 into free chunks, then B's release + a new deflate on s2 reuses
    # A's freed host slots: the new copy-out must wait for the copy-in that reads them
    pool.release(1, s2.cuda_stream)
    rc, ids_back = pool.inflate(slots, s1.cuda_stream)
    assert rc == 0
    assert pool.reserve([1], [wl.context], s2.cuda_stream) == 0
    _fill(pool, wl, 1, wl.context, s2)
    rc, slots_b = pool.deflate(pool.table(1)[0].tolist(), s2.cuda_stream)
    assert rc == 0 and sorted(slots_b.tolist()) == sorted(slots.tolist())
    torch.cuda.synchronize()
    for i in (0, 1234, n_chunks - 1):
        _check_chunk(pool.read_chunk(int(ids_back[i])), wl, 0, i)
        _check_chunk(pool.read_host_slot(int(slots_b[i])), wl, 1, i)
    pool.close()


def test_side_context_copies_follow_the_callers_stream():
    """Swap mode 3 on ONE stream with no host synchronisation: the side context's copy-out must
    start after the appends queued before it, and the work queued after an inflate (an append
    into the same request, then a read-back) must wait for the copy-in."""
    import torch
    from inputs import workload as W
    from paper_2506_15155_b200 import ellm
    wl = W.Workload("streams3", 32, 32, 8, 128, 2, 16000, seed=11, needle=False)
    n_chunks = 1000
    pool = ellm.Pool(0, 32, 32, 8, 128, 16, n_chunks + 8, n_chunks + 8, 2, n_chunks + 1, n_chunks)
    assert pool.set_swap_mode(3) == 0, pool.last_cuda_error()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        assert pool.reserve([0], [wl.context], s.cuda_stream) == 0
        _fill(pool, wl, 0, wl.context, s)               # ~2 GiB of appends, still running
        rc, slots = pool.deflate(pool.table(0)[0].tolist(), s.cuda_stream)
        assert rc == 0
        rc, ids = pool.inflate(slots, s.cuda_stream)   # back into (other) chunks
        assert rc == 0
    s.synchronize()
    for i in (0, 500, n_chunks - 1):
        _check_chunk(pool.read_host_slot(int(slots[i])), wl, 0, i)   # copied out after the appends
        _check_chunk(pool.read_chunk(int(ids[i])), wl, 0, i)          # copied in before the read
    pool.close()


def test_upload_through_side_context_is_exact_and_stream_ordered():
    """ellm_upload stages host -> device copies through the side context's 256 MiB buffer: a
    300 MiB upload (two pieces) on one stream immediately followed by another upload on a second
    stream (which must wait for the first one's use of the buffer) lands both byte-exactly, and
    a kernel queued after the upload on its stream sees the data."""
    import torch
    from paper_2506_15155_b200 import ellm
    pool = ellm.Pool(0, 2, 8, 2, 128, 16, 64, 64, 2, 32, 0)
    n = 300 << 20
    g = torch.Generator().manual_seed(5)
    h1 = torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g).pin_memory()
    h2 = torch.randint(0, 256, (n // 3,), dtype=torch.uint8, generator=g).pin_memory()
    d1 = torch.zeros(n, dtype=torch.uint8, device="cuda")
    d2 = torch.zeros(n // 3, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    assert pool.upload(d1, h1, stream=s1.cuda_stream) == 0, pool.last_cuda_error()
    assert pool.upload(d2, h2, stream=s2.cuda_stream) == 0
    with torch.cuda.stream(s1):
        c1 = d1.sum(dtype=torch.int64)   # queued after the upload on s1
    torch.cuda.synchronize()
    assert torch.equal(d1.cpu(), h1) and torch.equal(d2.cpu(), h2)
    assert int(c1) == int(h1.sum(dtype=torch.int64))
    assert pool.upload(d1, h1, 0) == 0 and pool.upload(d1, h1, -1) == ellm.INVALID_ARG
    pool.close()

"""Full-size parity in bench.py's launch configuration: BASELINE.json configs[1] (LLaMA-3-8B
shape, 32 requests x 32768 tokens, 128 GiB of KV in 2 MiB chunks) prefilled through
ellm_kv_append, one decode step, attention for all 32 requests at every sampled layer.
The oracle recomputes sampled (request, layer) outputs one by one from the same generator;
sampled chunks are compared byte for byte with the generator's rows."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2_pool():
    import torch
    from inputs import workload as W
    import gc
    gc.collect()
    torch.cuda.empty_cache()  # earlier tests' pools and torch's cached blocks
    free, _ = torch.cuda.mem_get_info()
    wl = W.c2()
    need = wl.batch * wl.chunks_per_request * wl.chunk_bytes() + (6 << 30)
    if free < need:
        pytest.skip(f"needs {need >> 30} GiB free HBM, have {free >> 30}")
    pool = W.make_pool(wl, 0)
    W.prefill(pool, wl)
    lens = np.full(wl.batch, wl.context, np.int64)
    q, k, v = W.decode_inputs(wl, 0, lens)
    reqs = list(range(wl.batch))
    assert pool.reserve(reqs, [1] * wl.batch) == 0
    out = torch.empty((wl.n_layers, wl.batch, wl.hq_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    for l in range(wl.n_layers):
        assert pool.append(l, reqs, [1] * wl.batch, k[l], v[l]) == 0
        assert pool.attention(l, reqs, q[l], out[l], 1.0 / np.sqrt(wl.head_dim)) == 0
    torch.cuda.synchronize()
    yield wl, pool, out
    pool.close()


@pytest.mark.parametrize("r,l", [(0, 0), (17, 31), (31, 0), (31, 31)])
def test_c2_sampled_attention(c2_pool, r, l):
    import oracle
    from inputs import workload as W
    from tests.twin import check_attention, torch_to_bits
    wl, pool, out = c2_pool
    k, v = W.host_kv(wl, r, l, wl.context + 1)
    ref = oracle.attention_contig(W.host_q(wl, r, l), k, v, 1.0 / np.sqrt(wl.head_dim))
    check_attention(torch_to_bits(out[l, r])[None], ref[None], f"C2 r={r} l={l}")


def test_c2_sampled_chunk_bytes(c2_pool):
    from inputs import gen
    wl, pool, _ = c2_pool
    T, L, Hkv, d = wl.tokens_per_chunk, wl.n_layers, wl.hkv_local, wl.head_dim
    for r, i in [(0, 0), (17, 1000), (31, 2047), (5, 2048)]:
        tab, ln = pool.table(r)
        assert ln == wl.context + 1 and len(tab) == 2049
        img = pool.read_chunk(int(tab[i])).view(np.uint16).reshape(L, 2, Hkv, T, d)
        rows = min(T, ln - i * T)
        pos = np.arange(i * T, i * T + rows)
        for l in (0, 13, 31):
            for kv in (0, 1):
                want = gen.kv_bits(wl.seed, r, pos, l, kv, range(Hkv), d, wl.group, wl.needle_range)
                assert np.array_equal(img[l, kv, :, :rows].transpose(1, 0, 2), want), (r, i, l, kv)

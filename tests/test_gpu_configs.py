"""Parity at the other BASELINE.json configs (full per-request sizes, sampled outputs):
C4 (LLaMA-70B shape, group 8, 10 MiB chunks) unsharded and as KV-head shards, C2 as a shard,
and C3 (8B-262K shape: 128K-token contexts) with swap-out / swap-in under memory pressure."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _decode_and_check(wl, samples, batch_check=True):
    import torch
    import oracle
    from inputs import workload as W
    from tests.twin import check_attention, torch_to_bits
    import gc
    gc.collect()
    torch.cuda.empty_cache()  # earlier tests' pools and torch's cached blocks
    free, _ = torch.cuda.mem_get_info()
    need = wl.batch * wl.chunks_per_request * wl.chunk_bytes() + (6 << 30)
    if free < need:
        pytest.skip(f"needs {need >> 30} GiB free HBM, have {free >> 30}")
    pool = W.make_pool(wl, 0)
    try:
        W.prefill(pool, wl)
        lens = np.full(wl.batch, wl.context, np.int64)
        q, k, v = W.decode_inputs(wl, 0, lens)
        reqs = list(range(wl.batch))
        assert pool.reserve(reqs, [1] * wl.batch) == 0
        out = torch.empty((wl.n_layers, wl.batch, wl.hq_local, wl.head_dim), dtype=torch.bfloat16,
                          device="cuda")
        for l in range(wl.n_layers):
            assert pool.append(l, reqs, [1] * wl.batch, k[l], v[l]) == 0
            assert pool.attention(l, reqs, q[l], out[l], 1.0 / np.sqrt(wl.head_dim)) == 0
        torch.cuda.synchronize()
        for r, l in samples:
            kk, vv = W.host_kv(wl, r, l, wl.context + 1)
            ref = oracle.attention_contig(W.host_q(wl, r, l), kk, vv, 1.0 / np.sqrt(wl.head_dim))
            check_attention(torch_to_bits(out[l, r])[None], ref[None], f"{wl.name} w{wl.world}r{wl.rank} r={r} l={l}")
    finally:
        pool.close()
        torch.cuda.synchronize()


def test_c4_single_gpu_batch32():
    from inputs import workload as W
    _decode_and_check(W.c4(batch=32), [(0, 0), (31, 79), (13, 40)])


@pytest.mark.parametrize("world,rank", [(2, 1), (4, 2), (8, 5)])
def test_c4_kv_head_shard(world, rank):
    from inputs import workload as W
    _decode_and_check(W.c4(world, rank), [(0, 79), (63, 0)])


@pytest.mark.parametrize("world,rank", [(2, 0), (8, 7)])
def test_c2_kv_head_shard(world, rank):
    from inputs import workload as W
    _decode_and_check(W.c2(world, rank), [(5, 31), (30, 2)])


@pytest.mark.parametrize("mode", [0, 3])
def test_c3_128k_contexts_with_swap_under_pressure(mode):
    """8B-262K shape, 4 requests x 131072 tokens (64 GiB of KV) in a device pool that holds
    3 of them: request 3 is prefilled, swapped out (deflate) to make room, request 0 is
    swapped out, request 3 swapped back in (inflate into request 0's freed chunks), then
    decode attention of the resident set is checked against the oracle. mode 0: SM copy
    kernels; mode 3: copy engines, the 16 GiB inflate staged through the side context."""
    import torch
    import oracle
    from inputs import workload as W
    from tests.twin import check_attention, torch_to_bits
    from paper_2506_15155_b200 import ellm
    wl = W.Workload("c3-llama3-8b-262k", 32, 32, 8, 128, 4, 131072, seed=2, tokens_per_chunk=16,
                    decode_headroom=16)
    cpr = wl.chunks_per_request  # 8193
    pool = ellm.Pool(0, 32, 32, 8, 128, 16, 4 * cpr, 3 * cpr + 1, 4, cpr, cpr)
    try:
        assert pool.set_swap_mode(mode) == 0
        s = torch.cuda.current_stream().cuda_stream
        # prefill requests 0..2, then free room for request 3 by deflating request 2's chunks
        sub = W.Workload(**{**wl.__dict__, "batch": 3})
        W.prefill(pool, sub)
        tab2 = pool.table(2)[0]
        rc, slots2 = pool.deflate(tab2, s)
        assert rc == 0
        # request 3 (its own prefill through the same append path)
        assert pool.reserve([3], [wl.context], s) == 0
        kbuf = torch.empty((wl.context, 8, 128), dtype=torch.bfloat16, device="cuda")
        vbuf = torch.empty_like(kbuf)
        for l in range(wl.n_layers):
            W.gen_kv_device(wl, 3, 0, wl.context, l, 0, kbuf.data_ptr(), s)
            W.gen_kv_device(wl, 3, 0, wl.context, l, 1, vbuf.data_ptr(), s)
            assert pool.append(l, [3], [wl.context], kbuf, vbuf, s) == 0
        del kbuf, vbuf
        assert pool.attention(0, [2], torch.empty(1, 32, 128, dtype=torch.bfloat16, device="cuda"),
                              torch.empty(1, 32, 128, dtype=torch.bfloat16, device="cuda"), 0.1, s) == ellm.NOT_RESIDENT
        # swap request 0 out, request 2 back in (into request 0's chunks)
        rc, slots0 = pool.deflate(pool.table(0)[0], s)
        assert rc == ellm.HOST_FULL  # host buffer holds one request: deflate is all-or-nothing
        rc = pool.release(0, s)
        assert rc == 0
        rc, ids2 = pool.inflate(slots2, s)
        assert rc == 0
        assert pool.stats()["host_used"] == 0
        torch.cuda.synchronize()
        reqs = [1, 2, 3]
        q = torch.empty((len(reqs), 32, 128), dtype=torch.bfloat16, device="cuda")
        out = torch.empty_like(q)
        for l in (0, 31):
            for i, r in enumerate(reqs):
                W.gen_q_device(wl, r, l, q[i].data_ptr(), s)
            assert pool.attention(l, reqs, q, out, 1.0 / np.sqrt(128), s) == 0
            torch.cuda.synchronize()
            for i, r in enumerate(reqs):
                kk, vv = W.host_kv(wl, r, l, wl.context)
                ref = oracle.attention_contig(W.host_q(wl, r, l), kk, vv, 1.0 / np.sqrt(128))
                check_attention(torch_to_bits(out[i])[None], ref[None], f"C3 r={r} l={l}")
    finally:
        pool.close()

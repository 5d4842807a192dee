"""f4 chunked prefill at full BASELINE.json sizes: a 2048-token prefill slab (C5's slab) at the
end of 32K-token contexts of the LLaMA-3-8B shape (configs[1] geometry) and at the end of 8K
contexts of the 70B shape (configs[3]: group 8, 10 MiB chunks with rotated slabs), two requests
per launch, in the kernel's production launch. Sampled query rows of every q-head are checked
against the definition the oracle's O12 follows: attention of position P over keys
0..P, i.e. oracle.attention_contig on the first P+1 generator rows, in fp64, within R8."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_Q = 2048


def _run(wl, layer, samples):
    import torch
    import oracle
    from inputs import gen
    from inputs import workload as W
    from tests.twin import bits_to_torch, check_attention, torch_to_bits
    import gc
    gc.collect()
    torch.cuda.empty_cache()  # earlier tests' pools and torch's cached blocks
    free, _ = torch.cuda.mem_get_info()
    need = wl.batch * wl.chunks_per_request * wl.chunk_bytes() + (4 << 30)
    if free < need:
        pytest.skip(f"needs {need >> 30} GiB free HBM, have {free >> 30}")
    pool = W.make_pool(wl, 0)
    try:
        W.prefill(pool, wl)  # every request holds `context` tokens of every layer
        B, Hq, d = wl.batch, wl.hq_local, wl.head_dim
        rng = np.random.default_rng(wl.seed + 101)
        q_bits = gen.f32_to_bf16(rng.standard_normal((B * N_Q, Hq, d)).astype(np.float32))
        out = torch.full((B * N_Q, Hq, d), float("nan"), dtype=torch.bfloat16, device="cuda")
        scale = 1.0 / np.sqrt(d)
        reqs = list(range(B))
        assert pool.prefill_attention(layer, reqs, [N_Q] * B, bits_to_torch(q_bits), out, scale) == 0
        torch.cuda.synchronize()
        got = torch_to_bits(out)
        for r in reqs:
            kk, vv = W.host_kv(wl, r, layer, wl.context)
            for k in samples:
                P = wl.context - N_Q + k  # absolute position of query k of request r
                ref = oracle.attention_contig(q_bits[r * N_Q + k], kk[:P + 1], vv[:P + 1], scale)
                check_attention(got[r * N_Q + k][None], ref[None], f"{wl.name} r={r} query {k} (pos {P})")
    finally:
        pool.close()
        torch.cuda.synchronize()


def test_prefill_slab_8b_shape_32k_context():
    from inputs import workload as W
    wl = W.c2()
    wl.batch = 2
    _run(wl, 17, [0, 1, 63, 64, 777, 1500, N_Q - 1])


def test_prefill_slab_70b_shape_rotated_slabs():
    from inputs import workload as W
    wl = W.c4(batch=2)
    _run(wl, 41, [0, 31, 32, 1024, N_Q - 1])

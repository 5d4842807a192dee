"""Parity of the exact launch sequence bench.py times, at full size (BASELINE.json configs[1]
and configs[3]): the pool is built and prefilled as bench.py builds it, launch overlap (PDL) is
on, and several decode steps run back to back with no host synchronisation — per step one
kv_reserve(+1) of every request, then per layer one ellm_decode_append_attention (new-token
append + attention + fused split-K merge). Only after the last step are sampled
(step, request, layer) outputs compared with the fp64 oracle (R8 tolerance) on the context that
step saw, and the chunks holding the decode-appended tokens compared bit for bit with the input
generator's rows."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STEPS = 4  # bench.py's warm-up (3) plus one timed step, all issued without a host sync


def _run(wl, samples, chunk_samples):
    import torch
    import oracle
    from inputs import gen
    from inputs import workload as W
    from tests.twin import check_attention, torch_to_bits
    import gc
    gc.collect()                 # pools of earlier tests in this process (their destructors free
    torch.cuda.empty_cache()     # the VMM memory) and torch's cached blocks
    free, _ = torch.cuda.mem_get_info()
    need = wl.batch * wl.chunks_per_request * wl.chunk_bytes() + (8 << 30)
    if free < need:
        pytest.skip(f"needs {need >> 30} GiB free HBM, have {free >> 30}")
    pool = W.make_pool(wl, 0)
    try:
        assert pool.set_launch_overlap(True) == 0
        W.prefill(pool, wl)
        L, B = wl.n_layers, wl.batch
        reqs, ones = list(range(B)), [1] * B
        lens = np.full(B, wl.context, np.int64)
        inputs = [W.decode_inputs(wl, s, lens + s) for s in range(STEPS)]
        out = torch.full((STEPS, L, B, wl.hq_local, wl.head_dim), float("nan"), dtype=torch.bfloat16,
                         device="cuda")
        sp = torch.cuda.current_stream().cuda_stream
        scale = 1.0 / np.sqrt(wl.head_dim)
        torch.cuda.synchronize()
        for s in range(STEPS):  # bench.py step(): no sync anywhere in the sequence
            q, k, v = inputs[s]
            assert pool.reserve(reqs, ones, sp) == 0
            for l in range(L):
                assert pool.decode_append_attention(l, reqs, k[l], v[l], q[l], out[s, l], scale, sp) == 0
        torch.cuda.synchronize()
        for s, r, l in samples:
            kk, vv = W.host_kv(wl, r, l, wl.context + s + 1)
            ref = oracle.attention_contig(W.host_q(wl, r, l), kk, vv, scale)
            check_attention(torch_to_bits(out[s, l, r])[None], ref[None], f"{wl.name} step={s} r={r} l={l}")
        # the chunks that received the STEPS decode tokens (and one prefill chunk) byte for byte
        T, Hkv, d = wl.tokens_per_chunk, wl.hkv_local, wl.head_dim
        final = wl.context + STEPS
        for r, i in chunk_samples:
            tab, ln = pool.table(r)
            assert ln == final and len(tab) == -(-final // T)
            img = pool.read_chunk(int(tab[i])).view(np.uint16).reshape(L, 2, Hkv, T, d)
            rows = min(T, ln - i * T)
            pos = np.arange(i * T, i * T + rows)
            for l in (0, L // 2, L - 1):
                for kv in (0, 1):
                    want = gen.kv_bits(wl.seed, r, pos, l, kv, range(wl.kv_head0, wl.kv_head0 + Hkv), d,
                                       wl.group, wl.needle_range)
                    assert np.array_equal(img[l, kv, :, :rows].transpose(1, 0, 2), want), (r, i, l, kv)
    finally:
        pool.close()
        torch.cuda.synchronize()


def test_c2_bench_sequence_full_size():
    """32 requests x 32768 tokens, 32 layers, fused decode launches with PDL, 4 steps."""
    from inputs import workload as W
    wl = W.c2()
    last = -(-(wl.context + STEPS) // wl.tokens_per_chunk) - 1
    _run(wl, [(0, 0, 0), (0, 31, 31), (1, 17, 5), (3, 31, 0), (3, 0, 31), (3, 12, 16)],
         [(0, last), (31, last), (17, 0), (9, last - 1)])


def test_c4_bench_sequence_full_size():
    """70B shape: 64 requests x 8192 tokens, 80 layers, 10 MiB chunks with rotated slabs."""
    from inputs import workload as W
    wl = W.c4()
    last = -(-(wl.context + STEPS) // wl.tokens_per_chunk) - 1
    _run(wl, [(0, 0, 79), (2, 63, 0), (3, 31, 40), (3, 5, 79)], [(0, last), (63, last), (40, 3)])

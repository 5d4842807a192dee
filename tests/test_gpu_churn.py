"""C5 churn (BASELINE.json configs[4]): 256 requests with log-uniform prompt lengths, mixed
prefill / decode, deflate / inflate under memory pressure, compaction by migration and
pool shrink / grow (tests/churn.py).

* scaled (lengths / 128, 2 layers): the oracle runs in lockstep (tests/twin.py) — every status
  code, table and stat bit-exact at every op, all live bytes at the end, sampled attention.
* full size (2K-128K prompts, LLaMA-3-8B geometry, 2 MiB chunks, device pool of 32 GiB +
  48 GiB pinned host slots): invariants that hold at any size after every iteration, sampled
  chunk bytes against the generator and sampled attention against the oracle.
"""
import numpy as np
import pytest

from tests.churn import Churn

pytestmark = pytest.mark.gpu


def test_c5_churn_scaled_lockstep_with_oracle():
    from tests.twin import Twin
    T, L = 16, 2
    t = Twin(L, 32, 8, 128, T, 160, 120, 256, 72, 640, seed=5)
    ch = Churn(t, 256, 2048 // 128, 131072 // 128, 8, 64, T, L, seed=5, slab=64, compact_every=16)

    def on_step(c, it):
        if it % 10 == 0:
            t.check_tables()
        if it % 25 == 0 and c.running:
            t.attention(it % L, c.running[:8])

    iters = ch.run(on_step=on_step)
    assert not ch.waiting and not ch.running and not ch.swapped, iters
    for k in ("admitted", "deflated", "inflated", "migrated", "grown", "shrunk", "released"):
        assert ch.stats[k] > 0, (k, ch.stats)
    t.check_tables()
    t.check_bytes()


class FullSide:
    """Product pool fed by the device-side generator (no oracle in lockstep)."""

    def __init__(self, wl, max_chunks, initial, host_slots):
        import torch
        from paper_2506_15155_b200 import ellm
        self.wl = wl
        self.p = ellm.Pool(0, wl.n_layers, wl.hq_local, wl.hkv_local, wl.head_dim, wl.tokens_per_chunk,
                           max_chunks, initial, wl.batch, wl.chunks_per_request, host_slots)
        self.lens = np.zeros(wl.batch, np.int64)
        self.kbuf = torch.empty((4096 * 4, wl.hkv_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
        self.vbuf = torch.empty_like(self.kbuf)
        self.s = torch.cuda.current_stream().cuda_stream

    def reserve(self, reqs, nn):
        rc = self.p.reserve(reqs, nn, self.s)
        if rc == 0:
            for r, n in zip(reqs, nn):
                self.lens[r] += n
        return rc

    def append_all_layers(self, reqs, nn):
        from inputs import workload as W
        row = self.wl.hkv_local * self.wl.head_dim * 2
        assert sum(nn) <= self.kbuf.shape[0]
        for l in range(self.wl.n_layers):
            off = 0
            for r, n in zip(reqs, nn):
                p0 = int(self.lens[r]) - n
                W.gen_kv_device(self.wl, r, p0, n, l, 0, self.kbuf.data_ptr() + off * row, self.s)
                W.gen_kv_device(self.wl, r, p0, n, l, 1, self.vbuf.data_ptr() + off * row, self.s)
                off += n
            assert self.p.append(l, reqs, nn, self.kbuf, self.vbuf, self.s) == 0

    def deflate(self, ids):
        return self.p.deflate(ids, self.s)

    def inflate(self, slots):
        return self.p.inflate(slots, self.s)

    def migrate(self, src, dst):
        return self.p.migrate(src, dst, self.s)

    def release(self, r):
        rc = self.p.release(r, self.s)
        if rc == 0:
            self.lens[r] = 0
        return rc

    def grow(self, n):
        return self.p.grow(n)

    def shrink(self, n):
        return self.p.shrink(n)


def check_invariants(side, n_requests):
    """I1-I3 and I6 from the product's own tables and chunk states."""
    st = side.p.stats()
    states = side.p.chunk_states()
    seen_c, seen_h = set(), set()
    for r in range(n_requests):
        tab, ln = side.p.table(r)
        assert ln == side.lens[r]
        assert len(tab) == (ln + side.wl.tokens_per_chunk - 1) // side.wl.tokens_per_chunk   # I1
        for e in tab.tolist():
            assert e != -1
            if e >= 0:
                assert e not in seen_c and states[e] == 1                                   # I2, I6
                seen_c.add(e)
            else:
                assert -e - 2 not in seen_h                                                  # I2
                seen_h.add(-e - 2)
    assert st["kv_used"] == len(seen_c) == int((states == 1).sum())                          # I6
    assert st["host_used"] == len(seen_h)
    assert st["kv_free"] + st["kv_used"] + st["act"] == len(states)                          # I3
    assert st["host_free"] + st["host_used"] == side.p.cfg.host_slots


def test_c5_churn_full_size():
    import torch
    import oracle
    from inputs import gen, workload as W
    from tests.twin import check_attention, torch_to_bits
    import gc
    gc.collect()
    torch.cuda.empty_cache()  # earlier tests' pools and torch's cached blocks
    free, _ = torch.cuda.mem_get_info()
    if free < (40 << 30):
        pytest.skip("needs 40 GiB free HBM")
    wl = W.Workload("c5-churn-8b", 32, 32, 8, 128, 256, 131072, seed=5, tokens_per_chunk=16,
                    decode_headroom=256, needle=False)
    side = FullSide(wl, max_chunks=16384, initial=12288, host_slots=24576)
    ch = Churn(side, 256, 2048, 131072, 16, 256, 16, 32, seed=5, slab=2048, compact_every=64)
    sampled = []

    def on_step(c, it):
        if it % 50 == 0:
            check_invariants(side, 256)
        if it % 200 == 100 and c.running:
            r = c.running[len(c.running) // 2]
            ln = int(side.lens[r])
            layer = it % 32
            q = torch.empty((1, 32, 128), dtype=torch.bfloat16, device="cuda")
            out = torch.empty_like(q)
            W.gen_q_device(wl, r, layer, q.data_ptr(), side.s)
            assert side.p.attention(layer, [r], q, out, 1 / np.sqrt(128), side.s) == 0
            torch.cuda.synchronize()
            kk, vv = W.host_kv(wl, r, layer, ln)
            ref = oracle.attention_contig(W.host_q(wl, r, layer), kk, vv, 1 / np.sqrt(128))
            check_attention(torch_to_bits(out[0])[None], ref[None], f"C5 it={it} r={r} len={ln}")
            tab, _ = side.p.table(r)
            i = len(tab) // 3
            if tab[i] >= 0:
                img = side.p.read_chunk(int(tab[i])).view(np.uint16).reshape(32, 2, 8, 16, 128)
                pos = np.arange(i * 16, i * 16 + 16)
                want = gen.kv_bits(wl.seed, r, pos, 5, 1, range(8), 128, 4, 0)
                assert np.array_equal(img[5, 1].transpose(1, 0, 2), want)
            sampled.append((it, r, ln))

    iters = ch.run(on_step=on_step)
    check_invariants(side, 256)
    assert not ch.waiting and not ch.running and not ch.swapped, (iters, ch.stats)
    assert len(sampled) >= 3
    for k in ("deflated", "inflated", "migrated", "grown", "shrunk"):
        assert ch.stats[k] > 0, (k, ch.stats)
    side.p.close()

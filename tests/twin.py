"""Test harness: the oracle and the CUDA path driven with identical operations and inputs.

Integer / byte state (tables, stats, status codes, chunk and host-slot bytes) must match
bit for bit; attention within BASELINE.json's tolerance (R8):
max |o - o_ref| <= 2e-2 and per (request, q-head) ||o - o_ref|| / ||o_ref|| <= 1e-2.
"""
from __future__ import annotations

import numpy as np

import oracle
from oracle import Oracle
from inputs import gen

ABS_TOL = 2e-2
REL_TOL = 1e-2


def bits_to_torch(a: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)


def torch_to_bits(t) -> np.ndarray:
    import torch
    return t.detach().view(torch.int16).cpu().numpy().view(np.uint16)


def check_attention(out_bits: np.ndarray, ref: np.ndarray, what=""):
    o = gen.bf16_to_f32(out_bits).astype(np.float64)
    err = np.abs(o - ref)
    assert np.isfinite(o).all(), f"{what}: non-finite output"
    assert err.max() <= ABS_TOL, f"{what}: max abs err {err.max():.3e}"
    num = np.linalg.norm(o - ref, axis=-1)
    den = np.maximum(np.linalg.norm(ref, axis=-1), 1e-30)
    rel = num / den
    assert rel.max() <= REL_TOL, f"{what}: max rel L2 err {rel.max():.3e}"
    return float(err.max()), float(rel.max())


class Twin:
    def __init__(self, L, Hq, Hkv, d, T, C, Ckv, R, MC, H, seed=0, needle=True, device=0,
                 q_head0=0, kv_head0=0, group=None, map_unit_bytes=0):
        from paper_2506_15155_b200 import ellm
        self.ellm = ellm
        self.o = Oracle(L, Hq, Hkv, d, T, C, Ckv, R, MC, H)
        self.p = ellm.Pool(device, L, Hq, Hkv, d, T, C, Ckv, R, MC, H, map_unit_bytes)
        self.L, self.Hq, self.Hkv, self.d, self.T, self.R = L, Hq, Hkv, d, T, R
        self.group = group or Hq // Hkv
        self.seed, self.needle = seed, needle
        self.q_head0, self.kv_head0 = q_head0, kv_head0
        self.lens = np.zeros(R, np.int64)
        self.scale = 1.0 / np.sqrt(d)

    # ---- ops ------------------------------------------------------------------------
    def reserve(self, reqs, nn):
        a, b = self.o.reserve(reqs, nn), self.p.reserve(reqs, nn)
        assert a == b, (a, b)
        if a == 0:
            for r, n in zip(reqs, nn):
                self.lens[r] += n
        return a

    def kv_rows(self, reqs, nn, layer):
        K, V = [], []
        heads = range(self.kv_head0, self.kv_head0 + self.Hkv)
        for r, n in zip(reqs, nn):
            pos = np.arange(self.lens[r] - n, self.lens[r])
            nr = int(self.lens[r]) if self.needle else 0
            K.append(gen.kv_bits(self.seed, r, pos, layer, 0, heads, self.d, self.group, nr))
            V.append(gen.kv_bits(self.seed, r, pos, layer, 1, heads, self.d, self.group, nr))
        return np.concatenate(K), np.concatenate(V)

    def append(self, layer, reqs, nn):
        K, V = self.kv_rows(reqs, nn, layer)
        a = self.o.append(layer, reqs, nn, K, V)
        b = self.p.append(layer, reqs, nn, bits_to_torch(K), bits_to_torch(V))
        assert a == b, (a, b)
        return a

    def append_all_layers(self, reqs, nn):
        for l in range(self.L):
            assert self.append(l, reqs, nn) == 0

    def q_bits(self, reqs, layer):
        heads = range(self.q_head0, self.q_head0 + self.Hq)
        return np.stack([gen.q_bits(self.seed + 7, r, layer, heads, self.d) for r in reqs])

    def attention(self, layer, reqs, check=True):
        import torch
        q = self.q_bits(reqs, layer)
        rc_o, ref = self.o.attention(layer, reqs, q, self.scale)
        out = torch.full((len(reqs), self.Hq, self.d), float("nan"), dtype=torch.bfloat16, device="cuda")
        rc_p = self.p.attention(layer, reqs, bits_to_torch(q), out, self.scale)
        torch.cuda.synchronize()
        assert rc_o == rc_p, (rc_o, rc_p)
        if rc_o != 0:
            return rc_o, None
        got = torch_to_bits(out)
        if check:
            check_attention(got, ref, f"layer {layer} reqs {list(reqs)[:8]}")
        return 0, (got, ref)

    def prefill_q_bits(self, layer, reqs, n_q, rng):
        """Queries for the last n_q positions of each request: N(0,1) rows, and on every other
        position each head carries 2x the key of a random visible position (a logit gap of
        ~2|k|^2/sqrt(d)), so a misplaced key or value moves the output by O(1). Needs needle=False
        (the keys are regenerated here from the counter-based generator)."""
        assert not self.needle
        heads = np.arange(self.kv_head0, self.kv_head0 + self.Hkv)
        out = []
        for r, m in zip(reqs, n_q):
            q = gen.f32_to_bf16(rng.standard_normal((m, self.Hq, self.d)).astype(np.float32))
            for k in range(0, m, 2):
                P = int(self.lens[r]) - m + k
                if P < 0:
                    break
                j = int(rng.integers(0, P + 1))
                kb = gen.kv_bits(self.seed, r, [j], layer, 0, heads, self.d, self.group, 0)[0]
                k2 = gen.f32_to_bf16(2.0 * gen.bf16_to_f32(kb))
                for h in range(self.Hq):
                    q[k, h] = k2[h // self.group]
            out.append(q)
        return np.concatenate(out)

    def prefill(self, layer, reqs, n_q, rng, check=True):
        """Causal chunked-prefill attention (f4): oracle O12 vs the tcgen05 kernel."""
        import torch
        q = self.prefill_q_bits(layer, reqs, n_q, rng)
        rc_o, ref = self.o.prefill_attention(layer, reqs, n_q, q, self.scale)
        out = torch.full((q.shape[0], self.Hq, self.d), float("nan"), dtype=torch.bfloat16, device="cuda")
        rc_p = self.p.prefill_attention(layer, reqs, n_q, bits_to_torch(q), out, self.scale)
        torch.cuda.synchronize()
        assert rc_o == rc_p, (rc_o, rc_p)
        if rc_o == 0 and check:
            return check_attention(torch_to_bits(out), ref, f"prefill layer {layer} reqs {list(reqs)[:8]}")
        return rc_o

    def decode_fused(self, layer, reqs):
        """Oracle: append of the pending token + attention; product: the fused single launch."""
        import torch
        K, V = self.kv_rows(reqs, [1] * len(reqs), layer)
        q = self.q_bits(reqs, layer)
        a = self.o.append(layer, reqs, [1] * len(reqs), K, V)
        rc_o, ref = self.o.attention(layer, reqs, q, self.scale) if a == 0 else (a, None)
        out = torch.full((len(reqs), self.Hq, self.d), float("nan"), dtype=torch.bfloat16, device="cuda")
        rc_p = self.p.decode_append_attention(layer, reqs, bits_to_torch(K), bits_to_torch(V),
                                              bits_to_torch(q), out, self.scale)
        torch.cuda.synchronize()
        assert rc_o == rc_p, (rc_o, rc_p)
        if rc_o == 0:
            check_attention(torch_to_bits(out), ref, f"fused layer {layer} reqs {list(reqs)[:8]}")
        return rc_o

    def deflate(self, ids):
        (a, sa), (b, sb) = self.o.deflate(ids), self.p.deflate(ids)
        assert a == b, (a, b)
        if a == 0:
            assert sa.tolist() == sb.tolist()
        return a, sa

    def inflate(self, slots):
        (a, sa), (b, sb) = self.o.inflate(slots), self.p.inflate(slots)
        assert a == b, (a, b)
        if a == 0:
            assert sa.tolist() == sb.tolist()
        return a, sa

    def migrate(self, src, dst):
        a, b = self.o.migrate(src, dst), self.p.migrate(src, dst)
        assert a == b, (a, b)
        return a

    def release(self, r):
        a, b = self.o.release(r), self.p.release(r)
        assert a == b
        if a == 0:
            self.lens[r] = 0
        return a

    def grow(self, n):
        a, b = self.o.grow(n), self.p.grow(n)
        assert a == b
        return a

    def shrink(self, n):
        a, b = self.o.shrink(n), self.p.shrink(n)
        assert a == b
        return a

    def act_alloc(self, n_chunks):
        a, b = self.o.act_alloc(n_chunks), self.p.act_alloc(n_chunks)
        assert a[0] == b[0] and (a[0] != 0 or a[1] == b[1]), (a, b)
        return a

    def act_free(self, first):
        a, b = self.o.act_free(first), self.p.act_free(first)
        assert a == b, (a, b)
        return a

    # ---- state checks ---------------------------------------------------------------
    def check_tables(self):
        for r in range(self.R):
            to, lo = self.o.table(r)
            tp, lp = self.p.table(r)
            assert lo == lp and to.tolist() == tp.tolist(), (r, to, tp)
        so, sp = self.o.stats(), self.p.stats()
        for k in so:
            assert so[k] == sp[k], (k, so, sp)

    def check_bytes(self):
        """Every live token row of every request, read through its table from the device chunk
        or pinned host slot, equals the oracle's image bit for bit."""
        import torch
        torch.cuda.synchronize()
        shape = (self.L, 2, self.Hkv, self.T, self.d)
        for r in range(self.R):
            tab, ln = self.o.table(r)
            for i, e in enumerate(tab.tolist()):
                rows = min(self.T, ln - i * self.T)
                if e >= 0:
                    a = self.o.read_chunk(e).view(np.uint16).reshape(shape)
                    b = self.p.read_chunk(e).view(np.uint16).reshape(shape)
                else:
                    h = -e - 2
                    a = self.o.read_host_slot(h).view(np.uint16).reshape(shape)
                    b = self.p.read_host_slot(h).view(np.uint16).reshape(shape)
                assert np.array_equal(a[:, :, :, :rows], b[:, :, :, :rows]), (r, i, e)

"""C5 serving loop (inputs/c5.py, the loop `bench.py --workload c5` times) run in lockstep with
the oracle: every product call the loop issues — chunked-prefill reserve / append / tcgen05
prefill attention, fused decode append + attention, offload (deflate), fetch (inflate),
compaction (migrate), pool grow / shrink, release — is mirrored on the oracle pool (O2-O9, O12)
with the same inputs. Status codes, tables and pool counters must match exactly and every
attention output must be within the R8 tolerance of the fp64 oracle."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class TeePool:
    """Forwards each call to the product pool and the oracle; checks they agree."""

    def __init__(self, p, o, Hq, d):
        self.p, self.o = p, o
        self.Hq, self.d = Hq, d
        self.chunk_bytes = p.chunk_bytes
        self.n_attn = 0

    def _same(self, a, b, what):
        assert a == b, (what, a, b)
        return a

    def stats(self):
        a, b = self.p.stats(), self.o.stats()
        for k in ("kv_free", "kv_used", "act", "host_free", "host_used"):
            assert a[k] == b[k], (k, a[k], b[k])
        return a

    def table(self, r):
        (ta, la), (tb, lb) = self.p.table(r), self.o.table(r)
        assert la == lb and np.array_equal(ta, tb), (r, ta, tb)
        return ta, la

    def chunk_states(self):
        return self.p.chunk_states()

    def kernel_launches(self):
        return self.p.kernel_launches()

    def grow(self, n):
        return self._same(self.p.grow(n), self.o.grow(n), "grow")

    def shrink(self, n):
        return self._same(self.p.shrink(n), self.o.shrink(n), "shrink")

    def reserve(self, reqs, nn, s):
        return self._same(self.p.reserve(reqs, nn, s), self.o.reserve(reqs, nn), "reserve")

    def append(self, layer, reqs, nn, k, v, s):
        from tests.twin import torch_to_bits
        m = int(sum(nn))
        rc = self.p.append(layer, reqs, nn, k, v, s)
        return self._same(rc, self.o.append(layer, reqs, nn, torch_to_bits(k[:m]), torch_to_bits(v[:m])), "append")

    def prefill_attention(self, layer, reqs, nq, q, out, scale, s):
        import torch
        from tests.twin import torch_to_bits, check_attention
        m = int(sum(nq))
        rc = self.p.prefill_attention(layer, reqs, nq, q, out, scale, s)
        rc2, ref = self.o.prefill_attention(layer, reqs, nq, torch_to_bits(q[:m]), scale)
        self._same(rc, rc2, "prefill_attention")
        torch.cuda.synchronize()
        check_attention(torch_to_bits(out[:m]), ref, f"c5 prefill layer {layer} reqs {reqs}")
        self.n_attn += 1
        return rc

    def decode_append_attention(self, layer, reqs, k, v, q, out, scale, s):
        import torch
        from tests.twin import torch_to_bits, check_attention
        n = len(reqs)
        rc = self.p.decode_append_attention(layer, reqs, k, v, q, out, scale, s)
        self._same(rc, self.o.append(layer, reqs, [1] * n, torch_to_bits(k[:n]), torch_to_bits(v[:n])), "append1")
        rc2, ref = self.o.attention(layer, reqs, torch_to_bits(q[:n]), scale)
        self._same(rc, rc2, "decode attention")
        torch.cuda.synchronize()
        check_attention(torch_to_bits(out[:n]), ref, f"c5 decode layer {layer}")
        self.n_attn += 1
        return rc

    def deflate(self, ids, s):
        (ra, sa), (rb, sb) = self.p.deflate(ids, s), self.o.deflate(ids)
        assert ra == rb and np.array_equal(sa, sb), (ra, rb, sa, sb)
        return ra, sa

    def inflate(self, slots, s):
        (ra, ca), (rb, cb) = self.p.inflate(slots, s), self.o.inflate(slots)
        assert ra == rb and np.array_equal(ca, cb), (ra, rb, ca, cb)
        return ra, ca

    def migrate(self, src, dst, s):
        return self._same(self.p.migrate(src, dst, s), self.o.migrate(src, dst), "migrate")

    def release(self, r, s):
        return self._same(self.p.release(r, s), self.o.release(r), "release")


@pytest.mark.timeout(900)
def test_c5_serve_loop_lockstep_with_oracle():
    import torch
    from oracle import Oracle
    from paper_2506_15155_b200 import ellm
    from inputs import workload as W
    from inputs.c5 import C5Serve, c5_lengths
    # 8B head geometry, 2 layers; prompts 64-3000 tokens, 256-token prefill slabs; a pool of
    # 320 x 16-token chunks (~5K tokens) against ~20K tokens of prompts: offload, fetch,
    # compaction and shrink / grow all happen within the run
    L, Hq, Hkv, d, T = 2, 32, 8, 128, 16
    n_req, C, C0, H = 24, 320, 240, 1024
    wl = W.Workload("c5-lockstep", L, Hq, Hkv, d, n_req, 3072, seed=5, tokens_per_chunk=T,
                    decode_headroom=64, needle=False)
    prompts, outs = c5_lengths(n_req, 5, 64, 3000, 4, 24)
    mc = wl.chunks_per_request
    p = ellm.Pool(0, L, Hq, Hkv, d, T, C, C0, n_req, mc, H)
    o = Oracle(L, Hq, Hkv, d, T, C, C0, n_req, mc, H)
    tee = TeePool(p, o, Hq, d)
    srv = C5Serve(tee, wl, prompts, outs, slab=256, compact_every=8, events=False)
    it = 0
    while (srv.waiting or srv.running or srv.swapped or srv.prefilling) and it < 3000:
        srv.step()
        it += 1
        if it % 5 == 0:
            tee.stats()
            for r in range(n_req):
                tee.table(r)
            assert o.check_invariants() == 0
    assert not srv.waiting and not srv.running and not srv.swapped and srv.prefilling is None, (it, srv.count)
    for k in ("deflated", "inflated", "migrated_chunks", "grown", "shrunk", "prefill_slabs", "decode_iters"):
        assert srv.count[k] > 0, (k, srv.count)
    assert tee.n_attn > 100
    st = tee.stats()
    assert st["kv_used"] == 0 and st["host_used"] == 0
    p.close()

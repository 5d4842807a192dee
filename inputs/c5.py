"""C5 serving loop (BASELINE.json configs[4]): mixed chunked-prefill / decode churn over a
device pool smaller than the working set, driven through libellm.so's own calls.

Harness policy only — the paper's Alg. 1 / Alg. 2 scheduling is out of scope;
this module holds no method arithmetic, it decides which product call runs next:

- FIFO admission with no hold-and-wait: a request is admitted only once the pool can
  hold its whole prompt (growing from ACT first, then offloading the least recently
  admitted running request to host slots);
- chunked prefill: the admitted request advances one `slab`-token chunk per iteration —
  kv_reserve(slab), then per layer kv_append + prefill_attention (f4) of that chunk;
- decode: every resident running request +1 token per iteration — kv_reserve(+1), then per
  layer one fused decode append + attention launch (rows a3-a5);
- offloaded requests are fetched back first when room exists, and admission
  waits while any are offloaded;
- finished requests release their chunks;
- every `compact_every` decode iterations the highest USED chunks are migrated to the lowest
  FREE ids (row a8) and half of the FREE chunks are returned to ACT (pool_shrink, row a9),
  re-grown on demand (pool_grow).

Every device call is bracketed by CUDA events on the stream it runs on, keyed by row, so the
bench can report sustained GB/s per row under churn. K/V/Q values are synthetic (the
seeded device generator, drawn once into per-layer buffers): this loop measures traffic;
parity of the same calls is what tests/ check.
"""
from __future__ import annotations

import numpy as np


class C5Serve:
    def __init__(self, pool, wl, prompts, outlens, slab=2048, compact_every=64, stream=None,
                 events=True, max_batch=None):
        import torch
        from inputs import workload as W
        self.p, self.wl = pool, wl
        self.T, self.L = wl.tokens_per_chunk, wl.n_layers
        self.prompt = np.asarray(prompts, np.int64)
        self.outlen = np.asarray(outlens, np.int64)
        n = len(self.prompt)
        self.slab, self.compact_every = slab, compact_every
        self.cs = stream or torch.cuda.current_stream()
        self.s = self.cs.cuda_stream
        self.waiting = list(range(n))
        self.prefilling = None      # [req, tokens done]
        self.running = []           # resident, decoding; admission order = LRU order
        self.swapped = []           # offloaded: (req, host slots)
        self.lens = np.zeros(n, np.int64)
        self.generated = np.zeros(n, np.int64)
        self.done = []
        self.scale = 1.0 / float(np.sqrt(wl.head_dim))
        self.events = events
        self.ev = []                # (row, start event, end event, algorithmic bytes or flops)
        self.count = {"admitted": 0, "prefill_slabs": 0, "prefill_tokens": 0, "decode_iters": 0,
                      "decode_tokens": 0, "deflated": 0, "deflated_chunks": 0, "inflated": 0,
                      "inflated_chunks": 0, "migrated_chunks": 0, "grown": 0, "shrunk": 0, "released": 0}
        Hq, Hkv, d, L = wl.hq_local, wl.hkv_local, wl.head_dim, self.L
        B = max_batch or n
        dev = "cuda"
        # synthetic inputs, drawn once: one prefill slab of K/V per layer (distinct buffers, so an
        # append never re-reads a source still in L2), one slab of Q, and a decode ring of B rows
        self.kslab = torch.empty((L, slab, Hkv, d), dtype=torch.bfloat16, device=dev)
        self.vslab = torch.empty_like(self.kslab)
        for layer in range(L):
            W.gen_kv_device(wl, 0, 0, slab, layer, 0, self.kslab[layer].data_ptr(), self.s)
            W.gen_kv_device(wl, 0, 0, slab, layer, 1, self.vslab[layer].data_ptr(), self.s)
        g = torch.Generator(device=dev)
        g.manual_seed(wl.seed)
        self.qslab = torch.randn((slab, Hq, d), device=dev, generator=g).to(torch.bfloat16)
        self.oslab = torch.empty_like(self.qslab)
        self.qd = torch.randn((L, B, Hq, d), device=dev, generator=g).to(torch.bfloat16)
        self.kd = torch.randn((L, B, Hkv, d), device=dev, generator=g).to(torch.bfloat16)
        self.vd = torch.randn((L, B, Hkv, d), device=dev, generator=g).to(torch.bfloat16)
        self.od = torch.empty_like(self.qd)
        self.host_io = None         # (pinned q, k, v, out) for end-to-end iterations
        torch.cuda.synchronize()

    # -- helpers ---------------------------------------------------------------------------
    def _ck(self, rc, what):
        if rc != 0:
            from paper_2506_15155_b200 import ellm
            raise ellm.EllmError(rc, what)

    def _chunks(self, n):
        return (int(n) + self.T - 1) // self.T

    def _timed(self, row, amount, fn):
        if not self.events:
            return fn()
        import torch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.cs)
        r = fn()
        e1.record(self.cs)
        self.ev.append((row, e0, e1, amount))
        return r

    def _st(self):
        return self.p.stats()

    def _deflate(self, r):
        ids = self.p.table(r)[0].tolist()
        if len(ids) > self._st()["host_free"]:
            return False
        rc, slots = self._timed("deflate", len(ids) * self.p.chunk_bytes, lambda: self.p.deflate(ids, self.s))
        self._ck(rc, "c5 deflate")
        self.running.remove(r)
        self.swapped.append((r, slots.tolist()))
        self.count["deflated"] += 1
        self.count["deflated_chunks"] += len(ids)
        return True

    def _make_room(self, need, protect=()):
        """Grow from ACT, else offload the least recently admitted unprotected running request."""
        while True:
            st = self._st()
            if st["kv_free"] >= need:
                return True
            grow = min(st["act"], need - st["kv_free"])
            if grow > 0:
                self._ck(self.p.grow(grow), "c5 grow")
                self.count["grown"] += grow
                continue
            victims = [r for r in self.running if r not in protect]
            if not victims or not self._deflate(victims[0]):
                return False

    # -- one scheduler iteration ---------------------------------------------------------
    def step(self, host=False):
        p, L = self.p, self.L
        # 1. fetch offloaded requests first
        while self.swapped:
            r, slots = self.swapped[0]
            st = self._st()
            if len(slots) > st["kv_free"] + st["act"] or not self._make_room(len(slots), protect=self.running):
                break
            rc, _ = self._timed("inflate", len(slots) * p.chunk_bytes, lambda: p.inflate(slots, self.s))
            self._ck(rc, "c5 inflate")
            self.swapped.pop(0)
            self.running.append(r)
            self.count["inflated"] += 1
            self.count["inflated_chunks"] += len(slots)
        # 2. FIFO admission (whole prompt must fit: no hold-and-wait)
        if self.prefilling is None and self.waiting and not self.swapped:
            r = self.waiting[0]
            if self._make_room(self._chunks(self.prompt[r]), protect=()):
                self.waiting.pop(0)
                self.prefilling = [r, 0]
                self.count["admitted"] += 1
        # 3. one chunked-prefill slab of the admitted request (append + causal attention, f4)
        if self.prefilling is not None:
            r, done = self.prefilling
            n = int(min(self.slab, self.prompt[r] - done))
            need = self._chunks(done + n) - self._chunks(done)
            if self._make_room(need, protect=(r,)):
                self._ck(p.reserve([r], [n], self.s), "c5 prefill reserve")
                self.lens[r] += n
                ctx = int(self.lens[r])
                Hkv, Hq, d = self.wl.hkv_local, self.wl.hq_local, self.wl.head_dim
                app_bytes = 2 * 2 * n * Hkv * d * 2                      # K,V read + write
                # causal QK^T + PV flops of n queries at positions ctx-n..ctx-1 (all q-heads)
                flops = 4 * Hq * d * (n * (ctx - n) + n * (n + 1) // 2)
                for layer in range(L):
                    self._ck(self._timed("prefill_append", app_bytes,
                                         lambda: p.append(layer, [r], [n], self.kslab[layer], self.vslab[layer],
                                                          self.s)), "c5 prefill append")
                    self._ck(self._timed("prefill_attn", flops,
                                         lambda: p.prefill_attention(layer, [r], [n], self.qslab, self.oslab,
                                                                     self.scale, self.s)), "c5 prefill attention")
                self.count["prefill_slabs"] += 1
                self.count["prefill_tokens"] += n
                done += n
                if done >= self.prompt[r]:
                    self.prefilling = None
                    self.running.append(r)
                else:
                    self.prefilling[1] = done
        # 4. decode +1 for every resident running request (fused append + attention per layer)
        if self.running:
            need = sum(1 for r in self.running if self.lens[r] % self.T == 0)
            prot = (self.prefilling[0],) if self.prefilling else ()
            self._make_room(need, protect=prot)
            reqs = list(self.running)
            if reqs and self._st()["kv_free"] >= sum(1 for r in reqs if self.lens[r] % self.T == 0):
                B = len(reqs)
                self._ck(p.reserve(reqs, [1] * B, self.s), "c5 decode reserve")
                self.lens[reqs] += 1
                Hkv, Hq, d = self.wl.hkv_local, self.wl.hq_local, self.wl.head_dim
                lens = self.lens[reqs]
                attn_bytes = (int(lens.sum()) * Hkv * d * 4 + 2 * B * Hq * d * 2
                              + 4 * int(sum(self._chunks(x) for x in lens)))
                qd, kd, vd, od = self.qd, self.kd, self.vd, self.od
                if host:
                    hq, hk, hv, ho = self.host_io
                    qd[:, :B].copy_(hq[:, :B], non_blocking=True)
                    kd[:, :B].copy_(hk[:, :B], non_blocking=True)
                    vd[:, :B].copy_(hv[:, :B], non_blocking=True)
                for layer in range(L):
                    self._ck(self._timed("decode_attn", attn_bytes,
                                         lambda: p.decode_append_attention(layer, reqs, kd[layer], vd[layer],
                                                                           qd[layer], od[layer], self.scale,
                                                                           self.s)), "c5 decode")
                if host:
                    ho[:, :B].copy_(od[:, :B], non_blocking=True)
                self.generated[reqs] += 1
                self.count["decode_iters"] += 1
                self.count["decode_tokens"] += B
                # 5. finished requests release their chunks
                for r in reqs:
                    if self.generated[r] >= self.outlen[r]:
                        self._ck(p.release(r, self.s), "c5 release")
                        self.running.remove(r)
                        self.done.append(r)
                        self.lens[r] = 0
                        self.count["released"] += 1
                # 6. compaction by migration + give half of the FREE chunks back (rows a8, a9)
                if self.count["decode_iters"] % self.compact_every == 0:
                    self.compact()

    def compact(self):
        p = self.p
        states = p.chunk_states()
        used = np.flatnonzero(states == 1)[::-1]
        free = np.flatnonzero(states == 0)
        k = 0
        while k < min(len(used), len(free)) and free[k] < used[k]:
            k += 1
        if k:
            src, dst = used[:k].tolist(), free[:k].tolist()
            self._ck(self._timed("migrate", 2 * k * p.chunk_bytes, lambda: p.migrate(src, dst, self.s)),
                     "c5 migrate")
            self.count["migrated_chunks"] += k
        n = self._st()["kv_free"] // 2
        if n:
            self._ck(p.shrink(n), "c5 shrink")
            self.count["shrunk"] += n

    def fast_fill(self):
        """Untimed setup: admit waiting requests by bulk append (no attention) while their whole
        prompt fits without offloading anything, so the timed loop starts under pressure."""
        p = self.p
        while self.waiting:
            r = self.waiting[0]
            st = self._st()
            if self._chunks(self.prompt[r]) + len(self.running) + 64 > st["kv_free"] + st["act"]:
                break
            self._make_room(self._chunks(self.prompt[r]))
            self.waiting.pop(0)
            left = int(self.prompt[r])
            while left > 0:
                n = min(self.slab, left)
                self._ck(p.reserve([r], [n], self.s), "fill reserve")
                self.lens[r] += n
                for layer in range(self.L):
                    self._ck(p.append(layer, [r], [n], self.kslab[layer], self.vslab[layer], self.s), "fill append")
                left -= n
            self.running.append(r)
            self.count["admitted"] += 1


def c5_lengths(n=256, seed=5, len_lo=2048, len_hi=131072, out_lo=16, out_hi=256):
    """BASELINE.json configs[4] length mix: prompts log-uniform in [2K, 128K], outputs uniform
    in [16, 256], seeded."""
    rng = np.random.default_rng(seed)
    prompts = np.exp(rng.uniform(np.log(len_lo), np.log(len_hi), n)).astype(np.int64)
    outs = rng.integers(out_lo, out_hi + 1, n)
    return prompts, outs

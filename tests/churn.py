"""C5 churn driver (BASELINE.json configs[4]): mixed prefill / decode with continuous append,
deflate / inflate and compaction by migration, over a device pool smaller than the working set.

Test-harness policy only (the paper's Alg. 1 is out of scope): FIFO admission with all of a
request's prefill chunks reserved at once per 2048-token slab (no hold-and-wait),
decode +1 token for every resident running request, least-recently-admitted request deflated
to host when chunks run short, swapped-out requests inflated back first when room exists,
and every `compact_every` steps the highest USED chunks are migrated to the lowest FREE ids and
half of the FREE chunks are returned (pool_shrink) to be re-grown on demand (pool_grow).

`side` is any object with the Twin API (tests/twin.py) — Twin itself (oracle + product in
lockstep) or FullSide (product only, device-generated inputs).
"""
from __future__ import annotations

import numpy as np


class Churn:
    def __init__(self, side, n_requests, len_lo, len_hi, out_lo, out_hi, T, n_layers, seed,
                 slab=2048, compact_every=64, host_slots=0):
        rng = np.random.default_rng(seed)
        self.side = side
        self.T = T
        self.L = n_layers
        self.slab = slab
        self.compact_every = compact_every
        self.prompt = np.exp(rng.uniform(np.log(len_lo), np.log(len_hi), n_requests)).astype(np.int64)
        self.outlen = rng.integers(out_lo, out_hi + 1, n_requests)
        self.waiting = list(range(n_requests))
        self.running = []          # resident, decoding (admission order = LRU order)
        self.swapped = []          # deflated: (req, slots)
        self.generated = np.zeros(n_requests, np.int64)
        self.done = []
        self.host_slots = host_slots
        self.stats = {"admitted": 0, "deflated": 0, "inflated": 0, "migrated": 0, "grown": 0,
                      "shrunk": 0, "decode_steps": 0, "prefill_slabs": 0, "released": 0}

    # helpers ---------------------------------------------------------------------------
    def _chunks(self, n):
        return (n + self.T - 1) // self.T

    def _free(self):
        return self.side.p.stats()["kv_free"]

    def _act(self):
        return self.side.p.stats()["act"]

    def _host_free(self):
        return self.side.p.stats()["host_free"]

    def _make_room(self, need, protect=()):
        """Grow from ACT, else deflate the least recently admitted running request."""
        while self._free() < need:
            grow = min(self._act(), need - self._free())
            if grow > 0:
                assert self.side.grow(grow) == 0
                self.stats["grown"] += grow
                continue
            victims = [r for r in self.running if r not in protect]
            if not victims:
                return False
            r = victims[0]
            ids = [int(c) for c in self.side.p.table(r)[0]]
            if len(ids) > self._host_free():
                return False
            rc, slots = self.side.deflate(ids)
            assert rc == 0, rc
            self.running.remove(r)
            self.swapped.append((r, slots))
            self.stats["deflated"] += 1
        return True

    # one scheduler iteration ------------------------------------------------------------
    def step(self):
        s = self.side
        # 1. resume swapped-out requests first (fetch when decoding is scheduled)
        while self.swapped:
            r, slots = self.swapped[0]
            if len(slots) > self._free() + self._act():
                break
            if not self._make_room(len(slots), protect=self.running):
                break
            rc, _ = s.inflate(slots)
            assert rc == 0, rc
            self.swapped.pop(0)
            self.running.append(r)
            self.stats["inflated"] += 1
        # 2. FIFO admission: one request per iteration, prefill slab by slab
        if self.waiting and not self.swapped:
            r = self.waiting[0]
            need = self._chunks(int(self.prompt[r]))
            if self._make_room(need, protect=()):
                self.waiting.pop(0)
                left = int(self.prompt[r])
                while left > 0:
                    n = min(self.slab, left)
                    assert s.reserve([r], [n]) == 0
                    s.append_all_layers([r], [n])
                    left -= n
                    self.stats["prefill_slabs"] += 1
                self.running.append(r)
                self.stats["admitted"] += 1
        # 3. decode +1 for resident running requests
        if self.running:
            reqs = list(self.running)
            need = sum(1 for r in reqs if s.lens[r] % self.T == 0)
            self._make_room(need, protect=())
            reqs = list(self.running)
            if reqs:
                rc = s.reserve(reqs, [1] * len(reqs))
                if rc == 0:
                    s.append_all_layers(reqs, [1] * len(reqs))
                    self.generated[reqs] += 1
                    self.stats["decode_steps"] += 1
        # 4. finished requests release their chunks
        for r in list(self.running):
            if self.generated[r] >= self.outlen[r]:
                assert s.release(r) == 0
                self.running.remove(r)
                self.done.append(r)
                self.stats["released"] += 1
        # 5. compaction + give half of the FREE chunks back
        if self.stats["decode_steps"] and self.stats["decode_steps"] % self.compact_every == 0:
            self.compact()

    def compact(self):
        s = self.side
        used = sorted(int(c) for r in self.running for c in s.p.table(r)[0])
        free = s.p.free_chunks()
        src, dst = [], []
        for a, b in zip(reversed(used), free):
            if b >= a:
                break
            src.append(a)
            dst.append(b)
        if src:
            assert s.migrate(src, dst) == 0
            self.stats["migrated"] += len(src)
        n = self._free() // 2
        if n:
            assert s.shrink(n) == 0
            self.stats["shrunk"] += n

    def run(self, max_iters=100000, on_step=None):
        it = 0
        while (self.waiting or self.running or self.swapped) and it < max_iters:
            self.step()
            if on_step:
                on_step(self, it)
            it += 1
        return it

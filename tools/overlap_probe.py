"""Why does decode slow down while a swap runs on a second stream? (DESIGN §5 open item.)

Decode steps of the C2 geometry (fused append+attention per layer) run on the compute stream
while one of several background loads runs on a second stream; the decode ms/step, the
background GB/s and nvidia-smi clocks/power during each phase are printed as one JSON line.
Not part of the product path; run on the box: python tools/overlap_probe.py [batch]."""
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


class Smi:
    F = ["clocks.sm", "clocks.mem", "power.draw", "clocks_event_reasons.sw_power_cap"]

    def __init__(self):
        self.lines = []

    def __enter__(self):
        self.p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=" + ",".join(self.F),
                                   "--format=csv,noheader,nounits", "-lms", "50"],
                                  stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        threading.Thread(target=lambda: [self.lines.append(x) for x in self.p.stdout], daemon=True).start()
        time.sleep(0.3)
        self.lines.clear()
        return self

    def __exit__(self, *a):
        self.p.terminate()

    def summary(self):
        sm, mem, pw, cap = [], [], [], 0
        for ln in self.lines:
            x = [s.strip() for s in ln.split(",")]
            try:
                sm.append(float(x[0])); mem.append(float(x[1])); pw.append(float(x[2]))
                cap += x[3].lower().startswith("active")
            except (ValueError, IndexError):
                pass
        if not sm:
            return {}
        return {"sm_mhz": float(np.median(sm)), "mem_mhz": float(np.median(mem)),
                "power_w": float(np.median(pw)), "power_cap_frac": round(cap / len(sm), 2), "n": len(sm)}


def main():
    from paper_2506_15155_b200 import ellm
    from inputs import workload as W
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    wl = W.c2()
    wl.batch = B
    swap_chunks = 1024
    pool = W.make_pool(wl, 0, host_slots=swap_chunks, extra_chunks=swap_chunks, extra_requests=1)
    W.prefill(pool, wl)
    W.fill_request(pool, wl, B, swap_chunks * 16)
    NB = int(sys.argv[2]) if len(sys.argv) > 2 else B  # requests that decode (footprint of the reads)
    reqs, ones = list(range(NB)), [1] * NB
    L = wl.n_layers
    scale = 1 / np.sqrt(128)
    lens = np.full(NB, wl.context, np.int64)
    NSTEP = 24
    wl_d = W.Workload(**{**wl.__dict__, "batch": NB})
    q, k, v = W.decode_inputs(wl_d, 0, lens)
    out = torch.empty((L, NB, 32, 128), dtype=torch.bfloat16, device="cuda")
    cs = torch.cuda.current_stream()
    sp = cs.cuda_stream

    def step():
        assert pool.reserve(reqs, ones, sp) == 0
        for l in range(L):
            assert pool.decode_append_attention(l, reqs, k[l], v[l], q[l], out[l], scale, sp) == 0

    N = 1 << 30
    hbuf = torch.empty(N, dtype=torch.uint8).pin_memory()
    dbuf = torch.empty(N, dtype=torch.uint8, device="cuda")
    dbuf2 = torch.empty(N, dtype=torch.uint8, device="cuda")
    ss = torch.cuda.Stream()
    ss2 = torch.cuda.Stream()
    # a THP-backed host buffer registered with cudaHostRegister (2 MiB host pages)
    import ctypes
    import mmap as _mm
    libc = ctypes.CDLL("libc.so.6", use_errno=True)
    libc.mmap.restype = ctypes.c_void_p
    libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
    thp = libc.mmap(None, N + (2 << 20), _mm.PROT_READ | _mm.PROT_WRITE, _mm.MAP_PRIVATE | _mm.MAP_ANONYMOUS, -1, 0)
    thp = (thp + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc.madvise(ctypes.c_void_p(thp), ctypes.c_size_t(N), 14)  # MADV_HUGEPAGE
    ctypes.memset(thp, 1, N)
    rc = torch.cuda.cudart().cudaHostRegister(thp, N, 0)
    print("thp register rc", rc, open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
          [l for l in open("/proc/meminfo") if l.startswith(("MemTotal", "MemAvailable", "AnonHugePages", "Hugepagesize"))],
          flush=True)

    def bg_thp(nrep, h2d=False):
        def go():
            for _ in range(nrep):
                if h2d:
                    assert ellm.memcpy_async(dbuf.data_ptr(), thp, N, ss) == 0
                else:
                    assert ellm.memcpy_async(thp, dbuf.data_ptr(), N, ss) == 0
            return N * nrep, ss
        return go

    SM = 64 << 20

    def bg_h2d_small(nrep, small_dst):
        def go():
            for _ in range(nrep):
                for j in range(N // SM):
                    if small_dst:
                        assert ellm.memcpy_async(dbuf.data_ptr(), hbuf.data_ptr() + j * SM, SM, ss) == 0
                    else:
                        assert ellm.memcpy_async(dbuf.data_ptr() + j * SM, hbuf.data_ptr(), SM, ss) == 0
            return N * nrep, ss
        return go

    def bg_mixed(in_mode, out_mode, nrep, h2d_gbs=0.0, d2h_gbs=0.0):
        def go():
            pool.set_swap_rate(h2d_gbs, d2h_gbs)
            moved = 0
            for _ in range(nrep):
                pool.set_swap_mode(out_mode)
                rc, slots = pool.deflate(pool.table(B)[0].tolist(), ss.cuda_stream)
                assert rc == 0
                pool.set_swap_mode(in_mode)
                rc, _ = pool.inflate(slots, ss.cuda_stream)
                assert rc == 0
                moved += 2 * len(slots) * pool.chunk_bytes
            return moved, ss
        return go

    def bg_memcpy(direction, nrep):
        def go():
            moved = 0
            for _ in range(nrep):
                with torch.cuda.stream(ss):
                    if direction == "d2h":
                        hbuf.copy_(dbuf, non_blocking=True)
                    else:
                        dbuf.copy_(hbuf, non_blocking=True)
                moved += N
            return moved, ss
        return go

    def bg_d2d(nrep):
        def go():
            for _ in range(nrep):
                with torch.cuda.stream(ss):
                    dbuf2.copy_(dbuf, non_blocking=True)
            return 2 * N * nrep, ss
        return go

    def bg_swap(mode, nrep):
        def go():
            pool.set_swap_mode(mode)
            moved = 0
            for _ in range(nrep):
                rc, slots = pool.deflate(pool.table(B)[0].tolist(), ss.cuda_stream)
                assert rc == 0
                rc, _ = pool.inflate(slots, ss.cuda_stream)
                assert rc == 0
                moved += 2 * len(slots) * pool.chunk_bytes
            return moved, ss
        return go

    def bg_bidir(nrep):
        def go():
            for _ in range(nrep):
                with torch.cuda.stream(ss):
                    hbuf.copy_(dbuf, non_blocking=True)
                with torch.cuda.stream(ss2):
                    dbuf2.copy_(hbuf, non_blocking=True)
            return 2 * N * nrep, ss
        return go

    rep = max(1, B // 16)
    phases = [("none", None), ("ce_h2d_contig", bg_memcpy("h2d", 16 * rep)), ("none_again", None)]
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    res = {"batch": B}
    for mode in ():  # isolated swap rates
        pool.set_swap_mode(mode)
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ss)
            moved, _ = bg_swap(mode, 1)()
            e1.record(ss)
            torch.cuda.synchronize()
        res[f"isolated_swap_mode{mode}_gbs"] = round(moved / e0.elapsed_time(e1) / 1e6, 2)
        print(f"isolated_swap_mode{mode}_gbs", res[f"isolated_swap_mode{mode}_gbs"], flush=True)
    for name, bg in phases:
        torch.cuda.synchronize()
        with Smi() as smi:
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record(cs)
            for _ in range(NSTEP):
                step()
            d1.record(cs)
            moved, bs = 0, None
            if bg is not None:
                s0.record(ss)
                moved, bs = bg()
                s1.record(ss)
            torch.cuda.synchronize()
        r = {"decode_ms_per_step": round(d0.elapsed_time(d1) / NSTEP, 3), **smi.summary()}
        if bg is not None:
            bms = s0.elapsed_time(s1)
            r["bg_gbs"] = round(moved / bms / 1e6, 2)
            r["bg_ms"] = round(bms, 1)
            r["decode_ms"] = round(d0.elapsed_time(d1), 1)
        res[name] = r
        print(name, r, flush=True)
    print(json.dumps(res))
    pool.close()


if __name__ == "__main__":
    main()

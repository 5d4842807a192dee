#!/usr/bin/env python
"""bench.py — decode-step throughput of the B200 eLLM KV-traffic hot path.

One step = one decode iteration of every request of the workload through the hot path
(SURVEY §8(a)): kv_reserve (+1 token each) and, for every layer, kv_append of the new
K/V, paged decode attention (+ split-K combine) and, for N > 1 GPUs, the all-gather of the
KV-head-sharded outputs. The elastic rows (deflate / inflate / migrate) are measured in
the same run as swap / migrate GB/s ("swap" object) against the host link measured there.

Default workload (N=1): BASELINE.json configs[1], LLaMA-3-8B shape (32 layers, 32q/8kv heads,
d=128), 32 requests x 32768 tokens of synthetic bf16 KV (128 GiB in 2 MiB chunks).
N > 1: the same workload KV-head-sharded over N GPUs (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ellm|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "tokens/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback (only if MEASURED_PEAKS.json absent)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default 40; c3: 4 swap rounds)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ellm", "reference"], default="ellm")
    ap.add_argument("--workload", choices=["c2", "c3", "c4", "c5"], default="c2",
                    help="c2 (default): 8B 32x32K; c3: 8B-262K 16x128K under memory pressure; c4: 70B 64x8K; "
                         "c5: 256-request prefill/decode churn with offload, compaction, shrink/grow")
    ap.add_argument("--swap-every", type=int, default=48,
                    help="c3: decode steps per offload/fetch round")
    ap.add_argument("--swap-mode", choices=["sm", "ce", "mixed", "staged", "ctx"], default="ctx",
                    help="c3: swap with the SM copy kernels, the DMA copy engines, copy engines for "
                         "swap-out and SM kernels for swap-in (mixed), copy engines with a staged "
                         "swap-in (host link -> staging buffer -> SM copy), or copy engines with the "
                         "swap-in through a second CUDA context's staging buffer (ctx, the default: "
                         "least interference with the decode, DESIGN.md §5 C3)")
    ap.add_argument("--c3-swapout", choices=["offload", "deflate"], default="offload",
                    help="c3: swap-out by layer-wise offload with the commit deferred until the copy "
                         "completed (default), or by deflate (frees the chunks at once, ordered after "
                         "the copy: the decode's next chunk allocation then waits for it)")
    ap.add_argument("--c3-offload-layers", type=int, default=2,
                    help="c3: layers of the swap-out enqueued per decode step (offload swap-out)")
    ap.add_argument("--resident", type=int, default=0,
                    help="c3: requests decoding in HBM (0 = as many as fit beside one in flight)")
    ap.add_argument("--gather", choices=["p2p", "nccl"], default="p2p",
                    help="N>1 head gather: fused into the attention epilogue over peer memory (p2p) "
                         "or a separate NCCL all-gather per layer")
    ap.add_argument("--batch", type=int, default=0,
                    help="override the workload's request count (testing; the JSON config records it)")
    ap.add_argument("--tokens-per-chunk", type=int, default=0,
                    help="override the workload's tokens per chunk T (layout study; the JSON config records it)")
    ap.add_argument("--layers", type=int, default=0, help="override the layer count (layout study)")
    ap.add_argument("--context", type=int, default=0, help="override the context length (layout study)")
    ap.add_argument("--emulate-shard", type=int, default=0,
                    help="run rank 0's shard of an N-way KV-head split alone on one GPU (no gather): the "
                         "per-GPU attention rate at the N-GPU geometry, for a box with fewer GPUs")
    ap.add_argument("--no-swap", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="wrap the timed steps in cudaProfilerStart/Stop (ncu --profile-from-start off)")
    a = ap.parse_args()
    if a.steps is None:
        a.steps = 4 * a.swap_every if a.workload == "c3" else 128 if a.workload == "c5" else 40
    return a


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def wait_first_sample(self, timeout=5.0):
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)
        self.lines.clear()

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def gpu_id_for(device: int) -> str:
    import torch
    try:
        p = torch.cuda.get_device_properties(device)
        return f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
    except Exception:
        return str(device)


# ----------------------------------------------------------------------------------------
# oracle legs (the only places bench.py executes oracle/)
# ----------------------------------------------------------------------------------------
def oracle_sample(wl, min_seconds=4.0):
    """Time the oracle (C++ fp64, OpenMP over q-heads, as it stands) on a bounded sample:
    attention of one request x one layer at the full context, repeated until >= min_seconds.
    Returns (seconds per request-layer, repeats, threads)."""
    import oracle
    from inputs import workload as W
    k, v = W.host_kv(wl, 0, 0, wl.context)
    q = W.host_q(wl, 0, 0)
    scale = 1.0 / (wl.head_dim ** 0.5)
    oracle.attention_contig(q, k[:16], v[:16], scale)  # load + warm
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.attention_contig(q, k, v, scale)
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds:
            break
    return el / reps, reps, oracle.num_threads()


def cpu_baseline_obj(wl, per_rl, reps, threads):
    tok_s = 1.0 / (wl.n_layers * per_rl)  # B requests x L layers per B tokens
    return {"value": round(tok_s, 4), "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": (f"oracle fp64 attention of 1 request x 1 layer at {wl.context} tokens "
                       f"({wl.hq_local} q-heads, {wl.hkv_local} kv-heads, d={wl.head_dim}) repeated {reps}x "
                       f"({per_rl:.3f} s each); extrapolated to {wl.batch} requests x {wl.n_layers} layers "
                       f"per decode step")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from inputs import workload as W
    import oracle
    if args.workload == "c5":
        print(json.dumps({"impl": "reference", "metric": METRIC,
                          "unavailable": "c5 is a churn schedule; the oracle arm is defined on c2/c3/c4"}), flush=True)
        return
    wl = {"c2": W.c2, "c3": W.c3, "c4": W.c4}[args.workload]()
    k, v = W.host_kv(wl, 0, 0, wl.context)
    q = W.host_q(wl, 0, 0)
    scale = 1.0 / (wl.head_dim ** 0.5)
    threads = oracle.num_threads()
    step_times = []
    for _ in range(args.warmup):
        oracle.attention_contig(q, k, v, scale)
    for _ in range(args.steps):  # each step: one request x one layer, scaled to the workload
        t0 = time.perf_counter()
        oracle.attention_contig(q, k, v, scale)
        step_times.append((time.perf_counter() - t0) * wl.n_layers * wl.batch)
    step = statistics.mean(step_times)
    value = wl.batch / step
    cb = cpu_baseline_obj(wl, step / (wl.n_layers * wl.batch), args.steps, threads)
    cb["value"] = round(value, 4)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based generator)",
        "config": workload_config(wl, args.gpus),
        "cpu_baseline": cb,
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("each step is a bounded sample: one request x one layer of the oracle, scaled to "
                 f"{wl.batch} requests x {wl.n_layers} layers"),
    }), flush=True)


def workload_config(wl, n):
    return {"workload": wl.name, "layers": wl.n_layers, "heads_q": wl.n_heads_q, "heads_kv": wl.n_heads_kv,
            "head_dim": wl.head_dim, "batch": wl.batch, "context": wl.context,
            "tokens_per_chunk": wl.tokens_per_chunk, "chunk_bytes": wl.chunk_bytes(),
            "parallelism": f"kv-head shard x{n}" if n > 1 else "single GPU",
            "l2": "inputs larger than L2 (KV read per layer >> 126 MB L2)"}


# ----------------------------------------------------------------------------------------
# the product leg
# ----------------------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "c3":
        return run_c3(args)
    if args.workload == "c5":
        return run_c5(args)
    import numpy as np
    import torch
    from paper_2506_15155_b200 import ellm
    from inputs import workload as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # ELLM_BENCH_SAME_GPU=1 (testing on a 1-GPU box): every rank on cuda:0, gloo process group;
    # the p2p gather then runs over CUDA IPC on one device instead of NVLink.
    same_gpu = os.environ.get("ELLM_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.emulate_shard > 1:
        if world > 1:
            raise SystemExit("--emulate-shard is a single-process mode")
        wl = W.c2(args.emulate_shard, 0) if args.workload == "c2" else W.c4(args.emulate_shard, 0)
    else:
        wl = W.c2(world, rank) if args.workload == "c2" else W.c4(world, rank)
    if args.batch:
        wl.batch = args.batch
    if args.tokens_per_chunk:
        wl.tokens_per_chunk = args.tokens_per_chunk
    if args.layers:
        wl.n_layers = args.layers
    if args.context:
        wl.context = args.context
    B, L = wl.batch, wl.n_layers
    swap_chunks = min(1024, wl.chunks_per_request) if not args.no_swap else 0
    t_create = time.perf_counter()
    # + one extra request (id = batch) of swap_chunks chunks: the swap / migrate measurements
    # move it between HBM and pinned host memory while the decode set stays resident
    pool = W.make_pool(wl, local, host_slots=swap_chunks, extra_chunks=swap_chunks,
                       extra_requests=1 if swap_chunks else 0)
    t_create = time.perf_counter() - t_create
    st_create = pool.stats()
    # the decode step issues the L attention launches back to back: let each overlap the
    # previous one's tail (PDL)
    pool.set_launch_overlap(True)
    prefill_appends = []
    W.prefill(pool, wl, append_times=prefill_appends)
    if swap_chunks:
        W.fill_request(pool, wl, wl.batch, swap_chunks * wl.tokens_per_chunk)
    reqs = list(range(B))
    ones = [1] * B
    scale = 1.0 / (wl.head_dim ** 0.5)
    lens = np.full(B, wl.context, np.int64)
    n_steps = args.warmup + args.steps
    e2e_steps = 0 if args.no_e2e else args.steps
    UNFUSED_STEPS = 3  # comparison: separate kv_append + attention launches
    CONC_STEPS = 45 if swap_chunks else 0  # decode steps with a concurrent swap stream (15 per mode)
    e2e_steps += CONC_STEPS
    e2e_steps += UNFUSED_STEPS
    # distinct per-step inputs in a ring capped at ~2 GiB (the 70B shape's 105 MB per step would
    # not fit beside its 165 GiB pool otherwise); values only feed traffic here, parity is tests/
    per_step = L * B * (wl.hq_local + 2 * wl.hkv_local) * wl.head_dim * 2
    n_ring = int(min(n_steps + e2e_steps, max(8, (2 << 30) // per_step)))

    class _Ring(list):
        def __getitem__(self, i):
            return list.__getitem__(self, i % len(self)) if isinstance(i, int) else list.__getitem__(self, i)

    inputs = _Ring()
    for s in range(n_ring):
        inputs.append(W.decode_inputs(wl, s, lens + s))
    out = torch.empty((L, B, wl.hq_local, wl.head_dim), dtype=torch.bfloat16, device="cuda")
    # --emulate-shard N issues rank 0's real N>1 call sequence (attention_gather + folded waits)
    # into a world-1 window: the per-GPU step minus the N-1 remote copies of each output row
    emulate = args.emulate_shard > 1
    p2p = (world > 1 or emulate) and args.gather == "p2p"
    gath = torch.empty((L, world, B, wl.hq_local, wl.head_dim), dtype=torch.bfloat16, device="cuda") \
        if world > 1 and not p2p else None
    pg = None
    if p2p:  # a10 fused: every rank's attention stores its heads' rows into all ranks' windows
        from paper_2506_15155_b200 import shard
        if emulate:
            pg = shard.PeerGather(pool, 1, 0, wl.hq_local, L, B, wl.head_dim, device=local)
        else:
            pg = shard.PeerGather(pool, world, rank, wl.n_heads_q, L, B, wl.head_dim, device=local)
            dist.barrier()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    attn_ev, app_ev, reserve_s = [], [], []

    def step(q, k, v, record=False, fused=True, o=None):
        o = out if o is None else o
        t0 = time.perf_counter()
        rc = pool.reserve(reqs, ones, sp)
        if record:
            reserve_s.append(time.perf_counter() - t0)
        if rc:
            raise ellm.EllmError(rc, "reserve")
        # fused: one event pair around the L back-to-back launches (an event between two
        # launches would keep the next from overlapping the previous one's tail, PDL), so the
        # per-launch time is the span / L; otherwise one pair per launch. With the p2p gather the
        # span includes the step's final gather_wait kernel.
        span = fused and gath is None
        for l in range(L):
            if fused:  # kv_append + attention + split-K merge in one launch per layer
                if record and (not span or l == 0):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                if pg is not None:  # ... + the head gather (a10) in the same launch
                    if l > 0:  # Q(l) needs every rank's rows of layer l-1: waited for inside
                        rc = pool.gather_wait_next(l - 1)  # this launch, after its first K/V TMAs
                        if rc:
                            raise ellm.EllmError(rc, "gather_wait_next")
                    rc = pool.attention_gather(l, reqs, q[l], pg.offset(l), scale, k[l], v[l], sp)
                else:
                    rc = pool.decode_append_attention(l, reqs, k[l], v[l], q[l], o[l], scale, sp)
                if rc:
                    raise ellm.EllmError(rc, "decode_append_attention")
            else:
                if record:
                    a0 = torch.cuda.Event(enable_timing=True)
                    a0.record(stream)
                rc = pool.append(l, reqs, ones, k[l], v[l], sp)
                if rc:
                    raise ellm.EllmError(rc, "append")
                if record:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    app_ev.append((a0, e0))
                if pg is not None:
                    rc = pool.attention_gather(l, reqs, q[l], pg.offset(l), scale, None, None, sp)
                else:
                    rc = pool.attention(l, reqs, q[l], o[l], scale, sp)
                if rc:
                    raise ellm.EllmError(rc, "attention")
            if pg is not None and (l == L - 1 or not fused):  # the step's result: every rank's rows
                rc = pool.gather_wait(l, sp)
                if rc:
                    raise ellm.EllmError(rc, "gather_wait")
            if record and (not span or l == L - 1):
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                attn_ev.append((e0, e1, L if span else 1))
            if gath is not None:
                dist.all_gather_into_tensor(gath[l], o[l])

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for s in range(args.warmup):
        step(*inputs[s])
    barrier()
    launches0 = pool.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_id_for(local)) as clk:
        clk.wait_first_sample()
        if args.profile:
            torch.cuda.profiler.start()
        ev0.record(stream)
        for s in range(args.warmup, n_steps):
            step(*inputs[s], record=True)
        ev1.record(stream)
        barrier()
        if args.profile:
            torch.cuda.profiler.stop()
    launches = pool.kernel_launches() - launches0
    el_ms = ev0.elapsed_time(ev1)
    attn_ms = [a.elapsed_time(b) / k for a, b, k in attn_ev]
    if dist:
        t = torch.tensor([el_ms, statistics.mean(attn_ms)], device="cpu" if same_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el_ms, attn_mean = float(t[0]), float(t[1])
    else:
        attn_mean = statistics.mean(attn_ms)
    ms_step = el_ms / args.steps
    value = B * args.steps / (el_ms / 1e3)

    # ---- roofline of the dominant kernel (paged attention + combine, one call per layer) ----
    lens_timed = lens + args.warmup + (args.steps + 1) / 2.0  # mean context during the timed steps
    T = wl.tokens_per_chunk
    alg_bytes = (wl.kv_bytes_per_layer(lens_timed) + 2 * B * wl.hq_local * wl.head_dim * 2
                 + 4 * int(sum(np.ceil(lens_timed / T))))
    achieved = alg_bytes / (attn_mean / 1e3) / 1e9
    peak, peak_src = hbm_peak()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if os.path.exists(tp) and world == 1 and not args.batch:  # captured for the N=1 workload only
        try:
            traffic = json.load(open(tp)).get(wl.name)
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": ("paged_attn_kernel: one ellm_decode_append_attention launch per layer (new-token "
                       "K/V append + attention + fused split-K merge)"),
            "alg_bytes_per_launch": int(alg_bytes), "launch_ms": round(attn_mean, 4), "peak_source": peak_src,
            "traffic_source": ("stored: dram__bytes_read.sum + dram__bytes_write.sum of one launch from the "
                               "committed ncu --set full capture (profiles/attn_traffic.json, same workload); "
                               "not measured in this run") if traffic is not None else None}

    # ---- end to end through host buffers: H2D of each step's inputs, D2H of its outputs ----
    e2e = None
    n_e2e = e2e_steps - UNFUSED_STEPS - CONC_STEPS
    if n_e2e:
        hin = _Ring()
        for s in range(n_steps, n_steps + min(n_e2e, n_ring)):
            hin.append(tuple(x.cpu().pin_memory() for x in inputs[s]))
        # Pipelined: step j+1's inputs are copied up on a second stream while step
        # j runs, and step j's result is read back on a third stream; inputs and outputs
        # double-buffered. (Measured, tools/e2e_probe.py: plain copies beat ellm_upload's
        # side-context staging here — these footprints / upload sizes see little interference.)
        dev_in = [tuple(torch.empty_like(x) for x in inputs[0]) for _ in range(2)]
        if pg is not None:  # the result of a step is the gathered [L, B, Hq, d] output
            hout = [torch.empty(L * pg.stride, dtype=torch.uint8).pin_memory() for _ in range(2)]
            outs = [out, out]  # the gather window is the output (one per rank, reused per step)
        else:
            hout = [torch.empty(out.shape, dtype=out.dtype).pin_memory() for _ in range(2)]
            outs = [out, torch.empty_like(out)]
        h2d = sum(x.numel() * x.element_size() for x in hin[0])
        d2h = hout[0].numel() * hout[0].element_size()
        up, dn = torch.cuda.Stream(), torch.cuda.Stream()
        ev_up, ev_used, ev_dl = [None, None], [None, None], [None, None]

        def upload(j):
            b = j % 2
            if ev_used[b] is not None:
                up.wait_event(ev_used[b])  # step j-2 has consumed this input set
            with torch.cuda.stream(up):
                for dt, ht in zip(dev_in[b], hin[j]):
                    dt.copy_(ht, non_blocking=True)
            ev_up[b] = torch.cuda.Event()
            ev_up[b].record(up)

        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        up.wait_event(e0)
        upload(0)
        for j in range(n_e2e):
            b = j % 2
            stream.wait_event(ev_up[b])
            if ev_dl[b] is not None and pg is None:
                stream.wait_event(ev_dl[b])  # step j-2's result has been read out of outs[b]
            step(*dev_in[b], o=outs[b])
            ev_used[b] = torch.cuda.Event()
            ev_used[b].record(stream)
            if j + 1 < n_e2e:
                upload(j + 1)
            dn.wait_event(ev_used[b])
            if pg is not None:  # the window is rewritten by the next step: read it on the compute stream
                ellm.memcpy_async(hout[b].data_ptr(), pg.out(0), d2h, sp)
            else:
                with torch.cuda.stream(dn):
                    hout[b].copy_(outs[b], non_blocking=True)
                ev_dl[b] = torch.cuda.Event()
                ev_dl[b].record(dn)
        stream.wait_stream(dn)
        e1.record(stream)
        barrier()
        ems = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ems], device="cpu" if same_gpu else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t[0])
        e2e = {"value": round(B * n_e2e / (ems / 1e3), 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ems / n_e2e, 3)}

    swap = measure_swap(pool, wl, stream) if swap_chunks else None

    # ---- swap overlapped with decode: the extra request is deflated / inflated on a second
    #      stream (3 rounds of 2 x 2 GiB) while CONC_STEPS decode steps run on the compute stream
    if swap_chunks:
        conc = {}
        c_first = n_steps + n_e2e
        for mi, (mode, name) in enumerate(((1, "ce"), (3, "ctx"), (0, "sm"))):
            pool.set_swap_mode(mode)
            ss = torch.cuda.Stream()
            barrier()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            half = CONC_STEPS // 3  # consecutive positions per mode
            base = c_first + mi * half
            d0.record(stream)  # decode first (the compute stream is busy ~half*20 ms) ...
            for s in range(base, base + half):
                step(*inputs[s])
            d1.record(stream)
            s0.record(ss)      # ... then the swap work, which overlaps it on the second stream
            moved = 0
            for _ in range(3):
                rc, slots = pool.deflate(pool.table(wl.batch)[0].tolist(), ss.cuda_stream)
                assert rc == ellm.OK, rc
                rc, _ = pool.inflate(slots, ss.cuda_stream)
                assert rc == ellm.OK, rc
                moved += 2 * len(slots) * pool.chunk_bytes
            s1.record(ss)
            barrier()
            swap_ms, dec_ms = s0.elapsed_time(s1), d0.elapsed_time(d1)
            conc[name] = {"decode_ms_per_step": round(dec_ms / half, 3), "swap_gbs": round(moved / swap_ms / 1e6, 2),
                          "swap_ms": round(swap_ms, 2), "decode_ms": round(dec_ms, 2)}
        pool.set_swap_mode(0)
        swap["concurrent_with_decode"] = {
            "isolated_decode_ms_per_step": round(ms_step, 4), **conc,
            "note": "3 rounds of deflate+inflate of 1024 x 2 MiB on a second stream during decode"}

    # ---- unfused comparison: the same step as separate kv_append and attention launches ----
    barrier()
    u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    u0.record(stream)
    for s in range(n_steps + e2e_steps - UNFUSED_STEPS, n_steps + e2e_steps):
        step(*inputs[s], record=True, fused=False)
    u1.record(stream)
    barrier()
    unfused_ms = u0.elapsed_time(u1) / UNFUSED_STEPS

    # ---- the other §8(a) rows: reserve (a2), append (a3), VMM create / grow / shrink (a1, a9) ----
    app_us = statistics.mean(a.elapsed_time(b) for a, b in app_ev) * 1e3
    bulk_s = sum(t for t, _ in prefill_appends)
    bulk_b = sum(nb for _, nb in prefill_appends)
    peak = hbm_peak()[0]
    st0 = pool.stats()
    n_vmm = min(256, st0["kv_free"])
    t0 = time.perf_counter()
    assert pool.shrink(n_vmm) == ellm.OK
    t_shrink = time.perf_counter() - t0
    t0 = time.perf_counter()
    assert pool.grow(n_vmm) == ellm.OK
    t_grow = time.perf_counter() - t0
    n_vmm = max(1, n_vmm)
    st1 = pool.stats()

    # ---- f1: the caller-side cost of shrink / grow of one default map unit while a
    #      decode step's attention launches are still queued on the GPU — device-synchronising
    #      unmap + on-demand map, vs asynchronous unmapping + speculative pre-mapping ----
    k_unit = min(max(1, (64 << 20) // pool.chunk_bytes), pool.stats()["kv_free"])

    def vmm_timed(fn):
        for l in range(L):
            pool.attention(l, reqs, inputs[0][0][l], out[l], scale, sp)
        s_before = pool.stats()
        t0 = time.perf_counter()
        assert fn() == ellm.OK
        dt = time.perf_counter() - t0
        s_after = pool.stats()
        torch.cuda.synchronize()
        assert pool.vmm_sync() == ellm.OK
        return {"host_ms": round(dt * 1e3, 3), "crit_vmm_ms": round((s_after["crit_vmm_ns"] - s_before["crit_vmm_ns"]) / 1e6, 3),
                "maps": s_after["n_map"] - s_before["n_map"], "unmaps": s_after["n_unmap"] - s_before["n_unmap"]}

    f1 = {"chunks": k_unit, "gpu_queue": f"{L} attention launches (~{ms_step:.0f} ms) queued before each call"}
    if k_unit == 0:
        f1["skipped"] = "no FREE chunks left in the pool"
    else:
        f1["sync"] = {"shrink": vmm_timed(lambda: pool.shrink(k_unit)), "grow": vmm_timed(lambda: pool.grow(k_unit))}
        assert pool.set_vmm_overlap(64 << 20, True) == ellm.OK and pool.vmm_sync() == ellm.OK
        f1["overlap"] = {"shrink": vmm_timed(lambda: pool.shrink(k_unit)), "grow": vmm_timed(lambda: pool.grow(k_unit)),
                         "premap_hits": pool.stats()["premap_hits"]}
        assert pool.set_vmm_overlap(0, False) == ellm.OK and pool.vmm_sync() == ellm.OK
    torch.cuda.synchronize()

    # ---- f4: chunked-prefill attention (tcgen05) over the same chunk-mapped KV: the last
    #      PF_NQ positions of PF_B requests attend causally to their whole context ----
    PF_B, PF_NQ, PF_ITERS = 4, 2048, 5
    pf_reqs = list(range(min(PF_B, B)))
    pf_len = [int(pool.table(r)[1]) for r in pf_reqs]
    qg = torch.Generator(device="cuda").manual_seed(11)
    pf_q = torch.randn((len(pf_reqs) * PF_NQ, wl.hq_local, wl.head_dim), generator=qg, device="cuda",
                       dtype=torch.bfloat16)
    pf_out = torch.empty_like(pf_q)
    assert pool.prefill_attention(0, pf_reqs, [PF_NQ] * len(pf_reqs), pf_q, pf_out, scale, sp) == ellm.OK
    p0e, p1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0e.record(stream)
    for it in range(PF_ITERS):
        pool.prefill_attention(it % L, pf_reqs, [PF_NQ] * len(pf_reqs), pf_q, pf_out, scale, sp)
    p1e.record(stream)
    torch.cuda.synchronize()
    pf_ms = p0e.elapsed_time(p1e) / PF_ITERS
    pf_keys = sum(sum(n - PF_NQ + i + 1 for i in range(PF_NQ)) for n in pf_len)
    pf_flops = 4.0 * wl.head_dim * pf_keys * wl.hq_local
    mp_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    bf16_peak = json.load(open(mp_path)).get("bf16_tflops") if os.path.exists(mp_path) else None
    f4 = {"requests": len(pf_reqs), "n_q": PF_NQ, "context": pf_len[0], "ms": round(pf_ms, 3),
          "tflops": round(pf_flops / pf_ms / 1e9, 1),
          "frac_of_bf16_peak": round(pf_flops / pf_ms / 1e9 / bf16_peak, 3) if bf16_peak else None,
          "flops": "4*d*sum_i(P_i+1)*Hq (causal, algorithmic)", "peak_source": "MEASURED_PEAKS.json bf16_tflops"}
    del pf_q, pf_out

    # ---- f2: layer-wise offload during prefill. The extra request (16K tokens) is
    #      prefilled layer by layer (one causal prefill-attention launch over all its positions per
    #      layer) with and without offloading each finished layer's slabs on a second stream; the
    #      exposed delay is what the O(N) offload adds to the O(N^2) prefill. Fetched back after. ----
    f2 = None
    if swap_chunks and world == 1:
        X = wl.batch
        ids = pool.table(X)[0].tolist()
        nX = int(pool.table(X)[1])
        nq = nX  # the whole request is prefilled (causal), layer by layer
        f2q = torch.randn((nq, wl.hq_local, wl.head_dim), generator=qg, device="cuda", dtype=torch.bfloat16)
        f2o = torch.empty_like(f2q)
        side = torch.cuda.Stream()

        def layers(offload):
            torch.cuda.synchronize()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            if offload:
                side.wait_event(c0)
                s0.record(side)
            for l in range(L):
                assert pool.prefill_attention(l, [X], [nq], f2q, f2o, scale, sp) == ellm.OK
                if offload:
                    e = torch.cuda.Event()
                    e.record(stream)
                    side.wait_event(e)
                    assert pool.offload_layer(l, ids, side.cuda_stream) == ellm.OK
            if offload:
                s1.record(side)
                stream.wait_stream(side)
            c1.record(stream)
            torch.cuda.synchronize()
            return c0.elapsed_time(c1), (s0.elapsed_time(s1) if offload else 0.0)

        layers(False)  # warm
        t_compute, _ = layers(False)
        off_bytes = len(ids) * pool.chunk_bytes
        f2 = {"request_tokens": nX, "chunks": len(ids), "offload_bytes": off_bytes, "n_q_per_layer": nq,
              "compute_ms": round(t_compute, 3),
              "note": "offload of layer l (second stream) follows that layer's causal prefill attention over "
                      "the whole request; sm = SM copy kernel, ce = DMA copy engines"}
        for mode, name in ((0, "sm"), (1, "ce")):
            pool.set_swap_mode(mode)
            ids = pool.table(X)[0].tolist()
            rc, f2_slots = pool.offload_begin(ids)
            assert rc == ellm.OK, rc
            t_both, t_side = layers(True)
            assert pool.offload_commit(ids, sp) == ellm.OK
            rc, _ = pool.inflate([-e - 2 for e in pool.table(X)[0].tolist()], sp)  # host slot h is -(h+2)
            assert rc == ellm.OK, rc
            torch.cuda.synchronize()
            f2[name] = {"compute_plus_offload_ms": round(t_both, 3), "exposed_ms": round(t_both - t_compute, 3),
                        "offload_stream_ms": round(t_side, 3),
                        "offload_gbs": round(off_bytes / (t_side / 1e3) / 1e9, 2)}
        pool.set_swap_mode(0)
        del f2q, f2o

    rows = {
        "a1_pool_create": {"s": round(t_create, 3), "chunks_mapped": st_create["n_map"],
                           "map_us_per_chunk": round(st_create["map_ns"] / max(1, st_create["n_map"]) / 1e3, 2),
                           "mapped_gib": round(st_create["mapped_bytes"] / 2 ** 30, 2)},
        "a2_kv_reserve": {"host_us_per_call": round(statistics.mean(reserve_s) * 1e6, 2), "requests": B},
        "step_fused_vs_unfused_ms": {"fused": round(ms_step, 4), "unfused": round(unfused_ms, 4)},
        "a3_kv_append": {"decode_us_per_call_unfused": round(app_us, 2),
                         "decode_bytes_per_call": 2 * 2 * B * wl.hkv_local * wl.head_dim * 2,
                         "bulk_gbs": round(bulk_b / bulk_s / 1e9, 1), "bulk_frac": round(bulk_b / bulk_s / 1e9 / peak, 3),
                         "bulk_calls": len(prefill_appends), "bulk_bytes_per_call": int(bulk_b / len(prefill_appends))},
        "a9_pool_shrink_grow": {"chunks": n_vmm, "shrink_ms": round(t_shrink * 1e3, 2), "grow_ms": round(t_grow * 1e3, 2),
                                "unmap_us_per_chunk": round((st1["unmap_ns"] - st0["unmap_ns"]) / max(1, n_vmm) / 1e3, 2),
                                "map_us_per_chunk": round((st1["map_ns"] - st0["map_ns"]) / max(1, n_vmm) / 1e3, 2)},
        "f1_vmm_overlap": f1,
        "f4_prefill": f4,
        "f2_layerwise_offload": f2,
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        per_rl, reps, threads = oracle_sample(wl)
        cpu = cpu_baseline_obj(wl, per_rl, reps, threads)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded counter-based generator, 3 needles per request/layer/kv-head)",
                "config": {**workload_config(wl, world),
                           **({"parallelism": f"rank 0 of a kv-head shard x{args.emulate_shard}, run alone on "
                                              "1 GPU: per-GPU rate at that geometry, with rank 0's N>1 call "
                                              "sequence (gather into a world-1 window: the N-1 remote row "
                                              "copies over NVLink are not issued)"}
                              if args.emulate_shard > 1 else {}),
                           **({"gather": "fused attention epilogue, P2P stores into every rank's window; "
                                         "layer l's wait folded into layer l+1's launch, gather_wait after "
                                         "the last layer"
                               if pg is not None else "NCCL all_gather_into_tensor per layer"}
                              if world > 1 or args.emulate_shard > 1 else {})},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clk.summary(),
                "attention_gbs": round(achieved, 1), "attention_frac_of_peak": roof["frac"], "swap": swap,
                "rows": rows}
        print(json.dumps(line), flush=True)
    if pg is not None:
        barrier()  # no rank unmaps its peers' windows while one may still write
        pg.close()
        barrier()
    pool.close()
    if dist:
        dist.destroy_process_group()


def run_c3(args):
    """BASELINE.json configs[2]: LLaMA-3-8B-262K shape, batch 16 x 128K context, decode under
    memory pressure. 256 GiB of KV does not fit one B200, so the pool holds R + 1 requests'
    chunks: R decode (the resident set) and one region is in flight. Every `swap_every` steps
    the least recently admitted request of the set is offloaded (deflate) and the next
    host-resident request is fetched into the freed chunks (inflate), on a second stream
    so the swap overlaps the decode of the set; the fetched request joins the set
    at the next round. All 16 requests progress round-robin; value = tokens/s of the whole job
    (R per step) over exactly K timed steps, swaps included."""
    import numpy as np
    import torch
    from paper_2506_15155_b200 import ellm
    from inputs import workload as W
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"metric": METRIC, "unavailable": "c3 is a single-GPU configuration"}), flush=True)
        return
    torch.cuda.set_device(0)
    wl = W.c3()
    total, L, Hq, Hkv, d, T = wl.batch, wl.n_layers, wl.hq_local, wl.hkv_local, wl.head_dim, wl.tokens_per_chunk
    cpr = wl.chunks_per_request
    req_bytes = cpr * wl.chunk_bytes()
    free, _ = torch.cuda.mem_get_info()
    fit = min(total, int((free - (5 << 30)) // req_bytes)) - 1
    R = min(fit, args.resident) if args.resident else fit  # measured best (C3)
    if R < 1:
        raise SystemExit("c3: not enough free HBM for one resident request plus one in flight")
    regions = R + 1
    host_reqs = total - R
    avail = 0
    for ln in open("/proc/meminfo"):
        if ln.startswith("MemAvailable"):
            avail = int(ln.split()[1]) * 1024
    if host_reqs * req_bytes > avail - (24 << 30):
        raise SystemExit(f"c3 needs {host_reqs * req_bytes >> 30} GiB of pinned host memory, "
                         f"{avail >> 30} GiB available")
    t0 = time.perf_counter()
    pool = ellm.Pool(0, L, Hq, Hkv, d, T, regions * cpr, regions * cpr, total, cpr, host_reqs * cpr)
    t_create = time.perf_counter() - t0
    cs = torch.cuda.current_stream()
    sp = cs.cuda_stream
    out_mode = {"sm": 0, "ctx": 3}.get(args.swap_mode, 1)
    in_mode = {"ce": 1, "staged": 2, "ctx": 3}.get(args.swap_mode, 0)
    pool.set_swap_mode(out_mode)
    # placement: requests R+1.. are prefilled through the pool and offloaded; 0..R stay
    host_q = []
    for r in range(R + 1, total):
        W.fill_request(pool, wl, r, wl.context)
        rc, slots = pool.deflate(pool.table(r)[0].tolist(), sp)
        if rc:
            raise ellm.EllmError(rc, "c3 offload")
        host_q.append((r, slots))
    for r in range(R + 1):
        W.fill_request(pool, wl, r, wl.context)
    torch.cuda.synchronize()
    D = list(range(R))            # the decoding set, oldest first
    incoming, in_ev = R, None     # fetched request, joins D at the next round
    sw = torch.cuda.Stream()
    scale = 1.0 / (d ** 0.5)
    ones = [1] * R
    slot_wl = W.Workload(**{**wl.__dict__, "batch": R})
    NIN = 8  # input ring: Q / new K,V of the R decode slots for 8 steps (synthetic values)
    inputs = [W.decode_inputs(slot_wl, s, np.full(R, wl.context + s, np.int64)) for s in range(NIN)]
    out = torch.empty((L, R, Hq, d), dtype=torch.bfloat16, device="cuda")
    attn_ev, swap_ev, swap_bytes, swap_mid = [], [], [], []
    tokens = {r: 0 for r in range(total)}

    # Swap-out: by default the request's chunks are copied out with the layer-wise
    # offload calls (offload_begin / offload_layer; the chunks stay USED and readable) and only
    # committed — tables repointed to the host slots, chunks freed — once the copy has completed
    # (polled at step boundaries). A deflate frees them at once instead, ordered after its copy:
    # the decode's next kv_reserve then takes the lowest free chunk, one of those being copied
    # out, and the compute stream waits for the whole 16 GiB copy-out (stream-ordered reuse, R7).
    pending = None  # (x, ids, slots, e0, em): swap-out copy in flight, commit not yet issued
    offload_todo = []  # layers of the pending swap-out not yet enqueued

    def swap_in_next(x, slots, e0, em):
        nonlocal incoming, in_ev
        host_q.append((x, slots))
        y, yslots = host_q.pop(0)
        pool.set_swap_mode(in_mode)
        e2, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(sw)                          # swap-in starts
        rc, _ = pool.inflate(yslots, sw.cuda_stream)
        if rc:
            raise ellm.EllmError(rc, "c3 inflate")
        e1.record(sw)
        in_ev, incoming = e1, y
        swap_ev.append((e0, e1))
        swap_mid.append((em, e2))
        swap_bytes.append(2 * len(slots) * pool.chunk_bytes)

    def finish_swap_out(block=False):
        nonlocal pending
        if pending is not None and offload_todo:
            if not block:
                offload_some()
                return
            while offload_todo:
                offload_some()
        if pending is None or not (block or pending[4].query()):
            return
        x, ids, slots, e0, em = pending
        pending = None
        if block:
            em.synchronize()
        rc = pool.offload_commit(ids, sw.cuda_stream)
        if rc:
            raise ellm.EllmError(rc, "c3 offload_commit")
        swap_in_next(x, slots, e0, em)

    def transition():
        nonlocal incoming, in_ev, pending
        finish_swap_out(block=True)            # (the previous round's, if still open)
        ev = torch.cuda.Event()
        ev.record(cs)
        sw.wait_event(ev)                      # X's last attention reads are done
        x = D.pop(0)
        if in_ev is not None:
            cs.wait_event(in_ev)               # the fetched request's bytes have landed
        D.append(incoming)
        e0, em = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sw)
        ids = pool.table(x)[0].tolist()
        pool.set_swap_mode(out_mode)
        if args.c3_swapout == "deflate":
            rc, slots = pool.deflate(ids, sw.cuda_stream)
            if rc:
                raise ellm.EllmError(rc, "c3 deflate")
            em.record(sw)
            swap_in_next(x, slots, e0, em)
            return
        rc, slots = pool.offload_begin(ids)
        if rc:
            raise ellm.EllmError(rc, "c3 offload_begin")
        pending = (x, ids, slots, e0, em)
        offload_todo[:] = list(range(L))
        offload_some()

    def offload_some():
        # a few layers per decode step (P:392 layer-wise), not all 16 GiB at once: a step's own
        # small device -> host copies (read-back of its result) share the copy engines in FIFO
        # order and would otherwise wait behind the whole copy-out
        if not offload_todo:
            return
        x, ids, slots, e0, em = pending
        for _ in range(min(args.c3_offload_layers, len(offload_todo))):
            rc = pool.offload_layer(offload_todo.pop(0), ids, sw.cuda_stream)
            if rc:
                raise ellm.EllmError(rc, "c3 offload_layer")
        if not offload_todo:
            em.record(sw)                      # swap-out copy done

    step_end = []  # per-step end events: the host runs at most LOOKAHEAD steps ahead of the GPU
    LOOKAHEAD = 3

    def step(s, record=False, host=None, o=None):
        o = out if o is None else o
        if len(step_end) >= LOOKAHEAD:
            step_end.pop(0).synchronize()
        finish_swap_out()
        if s and s % args.swap_every == 0:
            transition()
        q, k, v = inputs[s % NIN] if host is None else host
        rc = pool.reserve(D, ones, sp)
        if rc:
            raise ellm.EllmError(rc, "c3 reserve")
        for r in D:
            tokens[r] += 1
        lens_now = [int(pool.table(r)[1]) for r in D] if record else None
        for l in range(L):
            if record:
                a0 = torch.cuda.Event(enable_timing=True)
                a0.record(cs)
            rc = pool.decode_append_attention(l, D, k[l], v[l], q[l], o[l], scale, sp)
            if rc:
                raise ellm.EllmError(rc, "c3 decode_append_attention")
            if record:
                a1 = torch.cuda.Event(enable_timing=True)
                a1.record(cs)
                attn_ev.append((a0, a1, lens_now))
        se = torch.cuda.Event()
        se.record(cs)
        step_end.append(se)

    s_glob = 0
    for _ in range(args.warmup):
        step(s_glob)
        s_glob += 1
    torch.cuda.synchronize()
    launches0 = pool.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_swaps0 = len(swap_ev)
    with ClockSampler(gpu_id_for(0)) as clk:
        clk.wait_first_sample()
        ev0.record(cs)
        for _ in range(args.steps):
            step(s_glob, record=True)
            s_glob += 1
        ev1.record(cs)
        torch.cuda.synchronize()
    launches = pool.kernel_launches() - launches0
    el_ms = ev0.elapsed_time(ev1)
    value = R * args.steps / (el_ms / 1e3)
    timed_swaps = swap_ev[n_swaps0:]
    swap_ms = [a.elapsed_time(b) for a, b in timed_swaps]
    swap_gbs = [nb / (ms / 1e3) / 1e9 for nb, ms in zip(swap_bytes[n_swaps0:], swap_ms)]
    attn_ms = [a.elapsed_time(b) for a, b, _ in attn_ev]
    alg = [sum(lens) * Hkv * d * 4 + 2 * R * Hq * d * 2 + 4 * sum((n + T - 1) // T for n in lens)
           for _, _, lens in attn_ev]
    # decode steps by what the swap stream was doing meanwhile (times relative to ev0): a step is
    # [first launch start, last launch end]; it counts as "out" / "in" if it overlaps a swap-out /
    # swap-in phase of a timed round by more than half its length
    phases = []
    for (a, b), (m, m2) in zip(timed_swaps, swap_mid[n_swaps0:]):
        t0, tm, tm2, t1 = ev0.elapsed_time(a), ev0.elapsed_time(m), ev0.elapsed_time(m2), ev0.elapsed_time(b)
        phases += [("out", t0, tm), ("in", tm2, t1)]
    by_phase = {"out": [], "in": [], "none": []}
    for j in range(0, len(attn_ev) - L + 1, L):
        s0, s1 = ev0.elapsed_time(attn_ev[j][0]), ev0.elapsed_time(attn_ev[j + L - 1][1])
        ph = "none"
        for nm, p0, p1 in phases:
            if min(s1, p1) - max(s0, p0) > 0.5 * (s1 - s0):
                ph = nm
        by_phase[ph].append(s1 - s0)
    attn_mean = statistics.mean(attn_ms)
    achieved = statistics.mean(alg) / (attn_mean / 1e3) / 1e9
    peak, peak_src = hbm_peak()

    # the same resident set without swapping (isolated decode), and end to end through host buffers
    finish_swap_out(block=True)  # no swap work left in flight for the isolated steps
    torch.cuda.synchronize()
    if in_ev is not None:
        in_ev.synchronize()
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_iso = min(args.swap_every - 1, 16)
    s_iso = (s_glob // args.swap_every) * args.swap_every + 1  # no transition inside
    i0.record(cs)
    for j in range(n_iso):
        step(s_iso + j)
    i1.record(cs)
    torch.cuda.synchronize()
    iso_ms = i0.elapsed_time(i1) / n_iso
    e2e = None
    if not args.no_e2e:
        n_e2e = args.swap_every  # one full round, its transition included
        hin = [tuple(x.cpu().pin_memory() for x in inputs[j % NIN]) for j in range(n_e2e)]
        # pipelined as in the C2 / C4 e2e: step j+1's inputs copied up on a second stream while
        # step j runs, step j's output read back on a third; double-buffered
        dev = [tuple(torch.empty_like(x) for x in inputs[0]) for _ in range(2)]
        outs = [out, torch.empty_like(out)]
        hout = [torch.empty(out.shape, dtype=out.dtype).pin_memory() for _ in range(2)]
        up, dn = torch.cuda.Stream(), torch.cuda.Stream()
        ev_up, ev_used, ev_dl = [None, None], [None, None], [None, None]

        def upload(j):
            b = j % 2
            if ev_used[b] is not None:
                up.wait_event(ev_used[b])
            with torch.cuda.stream(up):
                for dt, ht in zip(dev[b], hin[j]):
                    dt.copy_(ht, non_blocking=True)
            ev_up[b] = torch.cuda.Event()
            ev_up[b].record(up)

        s_e = ((s_glob + n_iso) // args.swap_every + 1) * args.swap_every
        step_ev, host_ms = [], []
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        up.wait_event(e0)
        upload(0)
        for j in range(n_e2e):
            b = j % 2
            cs.wait_event(ev_up[b])
            if ev_dl[b] is not None:
                cs.wait_event(ev_dl[b])
            t_host = time.perf_counter()
            step(s_e + j, host=dev[b], o=outs[b])
            host_ms.append((time.perf_counter() - t_host) * 1e3)
            ev_used[b] = torch.cuda.Event(enable_timing=True)
            ev_used[b].record(cs)
            step_ev.append(ev_used[b])
            if j + 1 < n_e2e:
                upload(j + 1)
            dn.wait_event(ev_used[b])
            with torch.cuda.stream(dn):
                hout[b].copy_(outs[b], non_blocking=True)
            ev_dl[b] = torch.cuda.Event()
            ev_dl[b].record(dn)
        cs.wait_stream(dn)
        e1.record(cs)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        e2e = {"value": round(R * n_e2e / (ems / 1e3), 3), "unit": UNIT,
               "h2d_bytes_per_step": int(sum(x.numel() * x.element_size() for x in hin[0])),
               "d2h_bytes_per_step": int(hout[0].numel() * hout[0].element_size()),
               "ms_per_step": round(ems / n_e2e, 3), "steps": n_e2e,
               "step_end_ms": [round(e0.elapsed_time(x), 1) for x in step_ev],
               "host_ms_per_step": [round(x, 1) for x in host_ms]}
    torch.cuda.synchronize()
    cpu = None
    if not args.no_cpu_baseline:
        per_rl, reps, threads = oracle_sample(wl)
        cpu = cpu_baseline_obj(wl, per_rl, reps, threads)
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(el_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded counter-based generator, 3 needles per request/layer/kv-head)",
            "config": {**workload_config(wl, 1), "resident_requests": R, "host_requests": total - R - 1,
                       "in_flight_requests": 1, "swap_every_steps": args.swap_every,
                       "swap_mode": args.swap_mode, "swap_out": args.c3_swapout, "pool_gib": round(regions * req_bytes / 2 ** 30, 1),
                       "host_slots_gib": round(host_reqs * req_bytes / 2 ** 30, 1)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": None,
                         "kernel": "paged_attn_kernel (ellm_decode_append_attention, one launch per layer)",
                         "alg_bytes_per_launch": int(statistics.mean(alg)), "launch_ms": round(attn_mean, 4),
                         "peak_source": peak_src},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
            "c3": {"isolated_decode_ms_per_step": round(iso_ms, 4),
                   "swap_overhead_frac": round(1 - iso_ms / (el_ms / args.steps), 4),
                   "swaps_timed": len(timed_swaps),
                   "decode_ms_per_step_by_swap_phase": {k: {"steps": len(v), "mean_ms": round(statistics.mean(v), 3) if v else None}
                                                        for k, v in by_phase.items()},
                   "swap_out_ms": [round(b - a, 1) for _, a, b in phases[0::2]],
                   "swap_in_ms": [round(b - a, 1) for _, a, b in phases[1::2]],
                   "swap_round_ms": [round(x, 1) for x in swap_ms],
                   "swap_gbs_bidir_serial": [round(x, 2) for x in swap_gbs],
                   "bytes_per_swap_round": swap_bytes[-1] if swap_bytes else 0,
                   "tokens_per_request": [tokens[r] for r in range(total)],
                   "pool_create_s": round(t_create, 2)}}
    print(json.dumps(line), flush=True)
    pool.close()


def run_c5(args):
    """BASELINE.json configs[4]: 256 requests of the 8B shape with prompts
    log-uniform in [2K, 128K] and 16-256 output tokens, served by a FIFO loop (inputs/c5.py)
    over a device pool smaller than the working set: chunked prefill (2048-token slabs: append +
    tcgen05 prefill attention), decode of every resident request (fused append + attention per
    layer), offload of the least recently admitted request under pressure and fetch-back,
    compaction by migration and pool shrink / grow every 64 decode iterations. A step = one
    scheduler iteration; value = decode tokens/s over exactly K timed iterations (everything
    the iterations issue is inside the timed region); the c5 object reports prefill tokens/s
    and the sustained GB/s of every row under churn (CUDA events around each call)."""
    import numpy as np
    import torch
    from paper_2506_15155_b200 import ellm
    from inputs import workload as W
    from inputs.c5 import C5Serve, c5_lengths
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"metric": METRIC, "unavailable": "c5 is a single-GPU configuration"}), flush=True)
        return
    torch.cuda.set_device(0)
    wl = W.c5()
    n = wl.batch if not args.batch else args.batch
    prompts, outs = c5_lengths(n, wl.seed)
    free, _ = torch.cuda.mem_get_info()
    cb = wl.chunk_bytes()
    max_chunks = int((free - (10 << 30)) // cb)
    initial = max_chunks * 3 // 4          # the rest is ACT, grown on demand (pool_grow)
    host_slots = (48 << 30) // cb
    t0 = time.perf_counter()
    pool = ellm.Pool(0, wl.n_layers, wl.hq_local, wl.hkv_local, wl.head_dim, wl.tokens_per_chunk,
                     max_chunks, initial, n, wl.chunks_per_request, host_slots)
    t_create = time.perf_counter() - t0
    pool.set_swap_mode(1)                  # copy engines for offload / fetch
    pool.set_vmm_overlap(64 << 20, True)   # f1: pre-mapping + asynchronous unmapping
    cs = torch.cuda.current_stream()
    srv = C5Serve(pool, wl, prompts, outs, slab=2048, compact_every=64, stream=cs)
    srv.fast_fill()
    torch.cuda.synchronize()
    filled = dict(admitted=srv.count["admitted"], resident_gib=round(pool.stats()["kv_used"] * cb / 2 ** 30, 1))
    for _ in range(args.warmup):
        srv.step()
    torch.cuda.synchronize()
    srv.ev.clear()
    c0 = dict(srv.count)
    launches0 = pool.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_id_for(0)) as clk:
        clk.wait_first_sample()
        ev0.record(cs)
        for _ in range(args.steps):
            srv.step()
        ev1.record(cs)
        torch.cuda.synchronize()
    launches = pool.kernel_launches() - launches0
    el_ms = ev0.elapsed_time(ev1)
    dc = {k: srv.count[k] - c0[k] for k in srv.count}
    value = dc["decode_tokens"] / (el_ms / 1e3)
    rows = {}
    for row, e0, e1, amt in srv.ev:
        ms = e0.elapsed_time(e1)
        r = rows.setdefault(row, {"calls": 0, "ms": 0.0, "amount": 0})
        r["calls"] += 1
        r["ms"] += ms
        r["amount"] += amt
    peak, peak_src = hbm_peak()
    bf16_peak = None
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    bf16_src = None
    if os.path.exists(mp):  # inside a long step: the sustained (power-capped) GEMM figure
        j = json.load(open(mp))
        bf16_peak = j.get("bf16_tflops_sustained") or j.get("bf16_tflops")
        bf16_src = "measured (MEASURED_PEAKS.json " + (
            "bf16_tflops_sustained)" if j.get("bf16_tflops_sustained") else "bf16_tflops)")
    rows_out = {}
    for row, r in rows.items():
        o = {"calls": r["calls"], "ms_total": round(r["ms"], 2), "share_of_step": round(r["ms"] / el_ms, 4)}
        if row == "prefill_attn":
            tf = r["amount"] / (r["ms"] / 1e3) / 1e12
            o.update(tflops=round(tf, 1), frac_of_bf16_peak=round(tf / bf16_peak, 4) if bf16_peak else None)
        else:
            gbs = r["amount"] / (r["ms"] / 1e3) / 1e9
            o.update(gbs=round(gbs, 1), bytes=int(r["amount"]))
            if row in ("deflate", "inflate"):
                o["bound"] = "host link"
            else:
                o["frac_of_hbm"] = round(gbs / peak, 4)
        rows_out[row] = o
    dom = max(rows, key=lambda k: rows[k]["ms"]) if rows else None
    if dom == "prefill_attn" and bf16_peak:
        a = rows[dom]["amount"] / rows[dom]["calls"] / (rows[dom]["ms"] / rows[dom]["calls"] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": round(a, 1), "peak": bf16_peak, "unit": "TFLOP/s",
                "frac": round(a / bf16_peak, 4), "traffic": None,
                "kernel": "prefill_kernel (ellm_prefill_attention, tcgen05; one launch per layer per slab)",
                "peak_source": bf16_src}
    else:
        r = rows["decode_attn"]
        a = r["amount"] / (r["ms"] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(a, 1), "peak": peak, "unit": "GB/s", "frac": round(a / peak, 4),
                "traffic": None, "kernel": "paged_attn_kernel (ellm_decode_append_attention, one launch per layer)",
                "alg_bytes_per_launch": int(r["amount"] / r["calls"]), "launch_ms": round(r["ms"] / r["calls"], 4),
                "peak_source": peak_src}
    # end to end: the same loop with each iteration's decode Q/K/V copied from pinned host memory
    # and the attention outputs copied back, inside the timed region
    e2e = None
    if not args.no_e2e and srv.running:
        B = srv.qd.shape[1]
        srv.host_io = tuple(torch.empty(x.shape, dtype=x.dtype).pin_memory()
                            for x in (srv.qd, srv.kd, srv.vd, srv.od))
        srv.events = False
        n_e2e = 32
        t_before = srv.count["decode_tokens"]
        row_b = [0, 0]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(cs)
        for _ in range(n_e2e):
            b0 = srv.count["decode_tokens"]
            srv.step(host=True)
            nb = srv.count["decode_tokens"] - b0
            row_b[0] += nb * wl.n_layers * (wl.hq_local + 2 * wl.hkv_local) * wl.head_dim * 2
            row_b[1] += nb * wl.n_layers * wl.hq_local * wl.head_dim * 2
        e1.record(cs)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        e2e = {"value": round((srv.count["decode_tokens"] - t_before) / (ems / 1e3), 3), "unit": UNIT,
               "h2d_bytes_per_step": int(row_b[0] / n_e2e), "d2h_bytes_per_step": int(row_b[1] / n_e2e),
               "ms_per_step": round(ems / n_e2e, 3), "steps": n_e2e, "max_batch_rows": B,
               "note": ("the churn state moves on: these are the 32 iterations after the timed window, "
                        "with their own running batch and prefill mix; compare ms_per_step and "
                        "decode tokens per iteration, not only tokens/s")}
    cpu = None
    mean_len = int(np.mean([srv.lens[r] for r in srv.running])) if srv.running else 32768
    if not args.no_cpu_baseline:
        swl = W.Workload(**{**wl.__dict__, "context": mean_len, "batch": 1})
        per_rl, reps, threads = oracle_sample(swl)
        cpu = {"value": round(1.0 / (wl.n_layers * per_rl), 4), "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": (f"oracle fp64 decode attention of 1 request x 1 layer at the timed window's mean running "
                          f"context ({mean_len} tokens) repeated {reps}x ({per_rl:.3f} s each); decode tokens/s "
                          f"extrapolated to {wl.n_layers} layers per token (prefill, swap and compaction excluded)")}
    st = pool.stats()
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(el_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded lengths; device-generated K/V/Q values)",
            "config": {**workload_config(wl, 1), "batch": n, "context": "prompts log-uniform 2048-131072, outputs 16-256",
                       "pool_max_gib": round(max_chunks * cb / 2 ** 30, 1),
                       "pool_initial_gib": round(initial * cb / 2 ** 30, 1),
                       "host_slots_gib": round(host_slots * cb / 2 ** 30, 1), "prefill_slab": 2048,
                       "compact_every": 64, "swap_mode": "ce", "vmm_overlap": "premap 64 MiB + async unmap"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "c5": {"decode_tokens_per_s": round(value, 1),
                   "prefill_tokens_per_s": round(dc["prefill_tokens"] / (el_ms / 1e3), 1),
                   "total_tokens_per_s": round((dc["prefill_tokens"] + dc["decode_tokens"]) / (el_ms / 1e3), 1),
                   "timed_counts": dc, "rows": rows_out, "dominant_row": dom,
                   "after_fill": filled, "mean_running_context": mean_len,
                   "running_at_end": len(srv.running), "offloaded_at_end": len(srv.swapped),
                   "pool_at_end": {k: st[k] for k in ("kv_free", "kv_used", "act", "host_free", "host_used")},
                   "pool_create_s": round(t_create, 2)}}
    print(json.dumps(line), flush=True)
    pool.close()


def measure_swap(pool, wl, stream):
    """deflate / inflate / migrate GB/s over 1024 chunks (2 GiB at 2 MiB chunks) with the SM
    copy kernels and with the DMA copy engines, against pinned 1 GiB cudaMemcpyAsync (the
    host-link roofline, measured here)."""
    import torch
    from paper_2506_15155_b200 import ellm
    n = pool.stats()["host_free"]
    cb = pool.chunk_bytes
    sp = stream.cuda_stream

    def timed(fn):
        # device time of the call: a sleep kernel holds the stream while the host enqueues the
        # call (index upload + kernel / copies), so the events bracket only its device work
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3, r

    res = {}
    for mode, name in ((0, "sm"), (1, "ce"), (3, "ctx")):
        pool.set_swap_mode(mode)
        best_d2h, best_h2d, best_mig = 0.0, 0.0, 0.0
        for _ in range(3):
            ids = pool.table(wl.batch)[0][:n].tolist()  # the extra (non-decoding) request
            t, (rc, slots) = timed(lambda: pool.deflate(ids, sp))
            assert rc == ellm.OK, rc
            best_d2h = max(best_d2h, n * cb / t / 1e9)
            src = pool.table(1)[0][:n].tolist()
            nm = len(src)
            t, rc = timed(lambda: pool.migrate(src, sorted(ids)[:nm], sp))
            assert rc == ellm.OK, rc
            best_mig = max(best_mig, 2 * nm * cb / t / 1e9)
            t, (rc, back) = timed(lambda: pool.inflate(slots, sp))
            assert rc == ellm.OK, rc
            best_h2d = max(best_h2d, n * cb / t / 1e9)
        res[name] = {"d2h_gbs": round(best_d2h, 2), "h2d_gbs": round(best_h2d, 2),
                     "migrate_gbs": round(best_mig, 1)}
    pool.set_swap_mode(0)
    # host-link roofline: pinned 1 GiB copies, best of 5
    N = 1 << 30
    h = torch.empty(N, dtype=torch.uint8).pin_memory()
    d = torch.empty(N, dtype=torch.uint8, device="cuda")
    link = {}
    for nm, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 0.0
        for _ in range(5):
            t, _ = timed(fn)
            best = max(best, N / t / 1e9)
        link[nm] = round(best, 2)
    best_sm = max(res["sm"]["d2h_gbs"] / link["d2h"], 0)
    return {"chunks": n, "chunk_bytes": cb, "bytes": n * cb, "modes": res, "link_gbs": link,
            "frac_d2h": round(max(res["sm"]["d2h_gbs"], res["ce"]["d2h_gbs"]) / link["d2h"], 3),
            "frac_h2d": round(max(res["sm"]["h2d_gbs"], res["ce"]["h2d_gbs"]) / link["h2d"], 3),
            "migrate_frac_of_hbm": round(max(res["sm"]["migrate_gbs"], res["ce"]["migrate_gbs"]) / hbm_peak()[0], 3),
            "_sm_d2h_frac": round(best_sm, 3)}


if __name__ == "__main__":
    main()

"""Library context for f4: the same causal prefill shapes as tools/prefill_bench.py (8B geometry,
Hq 32 / Hkv 8 / d 128, bf16; B requests whose last n_q positions attend causally to ctx keys)
timed with library attention kernels on contiguous K/V on this box:
  - torch SDPA, cuDNN backend (cuDNN's fused attention for sm_100)
  - torch SDPA, flash backend (FlashAttention-2 kernels built into torch)
  - flashinfer BatchPrefillWithRaggedKVCacheWrapper, backend "cutlass" (its sm_100 FMHA, JIT-built)
Each is skipped with the reason if it is unavailable for a shape. Same algorithmic flop count as
prefill_bench.py (4·d per visible (query, key) pair per q-head), CUDA events, 10 iterations after
2 warm-ups. Context only: none of these is on the product path.
  python tools/prefill_lib_compare.py [--no-flashinfer]"""
import sys
import time

import torch
import torch.nn.functional as F

SHAPES = [(1, 8192, 8192), (4, 4096, 4096), (8, 16384, 2048), (16, 2048, 2048), (2, 32768, 4096)]
Hq, Hkv, D = 32, 8, 128


def flops(B, ctx, nq):
    keys = sum(ctx - nq + i + 1 for i in range(nq))
    return 4.0 * D * keys * Hq * B


def timeit(fn, iters=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def sdpa(backend, B, ctx, nq):
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from torch.nn.attention.bias import causal_lower_right
    q = torch.randn(B, Hq, nq, D, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(B, Hq, ctx, D, device="cuda", dtype=torch.bfloat16)  # GQA expanded
    v = torch.randn(B, Hq, ctx, D, device="cuda", dtype=torch.bfloat16)
    be = {"cudnn": SDPBackend.CUDNN_ATTENTION, "flash": SDPBackend.FLASH_ATTENTION}[backend]
    if nq == ctx:
        f = lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True)  # noqa: E731
    else:
        m = causal_lower_right(nq, ctx)
        f = lambda: F.scaled_dot_product_attention(q, k, v, attn_mask=m)  # noqa: E731
    with sdpa_kernel([be]):
        return timeit(f)


def flashinfer_cutlass(B, ctx, nq):
    import flashinfer
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    w = flashinfer.prefill.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend="cutlass")
    qo = torch.arange(0, B + 1, dtype=torch.int32, device="cuda") * nq
    kv = torch.arange(0, B + 1, dtype=torch.int32, device="cuda") * ctx
    w.plan(qo, kv, Hq, Hkv, D, causal=True, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
    q = torch.randn(B * nq, Hq, D, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(B * ctx, Hkv, D, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(B * ctx, Hkv, D, device="cuda", dtype=torch.bfloat16)
    return timeit(lambda: w.run(q, k, v))


def main():
    impls = [("cudnn", lambda *s: sdpa("cudnn", *s)), ("torch-flash", lambda *s: sdpa("flash", *s))]
    if "--no-flashinfer" not in sys.argv:
        impls.append(("flashinfer-cutlass", flashinfer_cutlass))
    for name, fn in impls:
        for B, ctx, nq in SHAPES:
            t0 = time.time()
            try:
                ms = fn(B, ctx, nq)
                print(f"{name:18s} B={B} ctx={ctx} n_q={nq}: {ms:.3f} ms  {flops(B, ctx, nq) / ms / 1e9:.1f} TFLOP/s",
                      flush=True)
            except Exception as e:  # report and continue
                msg = str(e).strip().splitlines()[0][:160] if str(e).strip() else type(e).__name__
                print(f"{name:18s} B={B} ctx={ctx} n_q={nq}: unavailable ({type(e).__name__}: {msg}) "
                      f"[{time.time() - t0:.0f} s]", flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

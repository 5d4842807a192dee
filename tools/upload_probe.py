"""ellm_upload rate (host -> side-context staging -> device) vs a plain host -> device copy, from
torch-pinned and from portable pinned host memory; device-timed. python tools/upload_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402
from paper_2506_15155_b200 import ellm  # noqa: E402

pool = ellm.Pool(0, 2, 8, 2, 128, 16, 64, 64, 2, 32, 0)
n = 100 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
err, hp = cu.cuMemHostAlloc(n, cu.CU_MEMHOSTALLOC_PORTABLE)
s = torch.cuda.current_stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return f"{ms:.3f} ms  {n / ms / 1e6:.1f} GB/s"


print("torch copy_      ", timed(lambda: d.copy_(h, non_blocking=True)))
print("upload (torch pinned)   ", timed(lambda: pool.upload(d, h, stream=s.cuda_stream)))
print("upload (portable pinned)", timed(lambda: pool.upload(d, int(hp), n, stream=s.cuda_stream)))

"""Background host->device traffic in its own process (and CUDA context) for the two-process
interference probe (tools/interference_ncu.sh): pinned 1 GiB -> device copies back to back for
--seconds, then prints the achieved rate. Touches `--ready` once the first copy completed."""
import argparse
import time

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=300.0)
ap.add_argument("--ready", default="")
ap.add_argument("--kind", choices=["h2d", "d2h"], default="h2d")
a = ap.parse_args()
N = 1 << 30
h = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device="cuda")
t0, n = time.time(), 0
while time.time() - t0 < a.seconds:
    for _ in range(4):
        (d.copy_(h, non_blocking=True) if a.kind == "h2d" else h.copy_(d, non_blocking=True))
    torch.cuda.synchronize()
    n += 4
    if n == 4 and a.ready:
        open(a.ready, "w").close()
print(f"{a.kind}_loop: {n} GiB in {time.time() - t0:.1f} s = {n * N / (time.time() - t0) / 1e9:.1f} GB/s", flush=True)

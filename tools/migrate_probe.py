"""Migrate (a8) GB/s at the C2 (2 MiB chunks) and C4 (10 MiB, rotated slabs) geometries, TMA bulk
kernel vs warp copy kernel (ELLM_D2D_BULK), device time: the stream is held by a sleep kernel
while the call is enqueued, so the events bracket only the call's device work."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_15155_b200 import ellm  # noqa: E402
from inputs import workload as W  # noqa: E402


def run(wl, n_move, reps=5):
    pool = W.make_pool(wl, 0, extra_chunks=n_move, extra_requests=1)
    W.fill_request(pool, wl, 0, n_move * wl.tokens_per_chunk)
    s = torch.cuda.current_stream()
    out = {}
    for bulk in ("1", "0"):
        os.environ["ELLM_D2D_BULK"] = bulk
        best = 0.0
        for _ in range(reps):
            src = pool.table(0)[0].tolist()
            free = sorted(set(range(pool.stats()["kv_free"] + pool.stats()["kv_used"])) - set(src))[:n_move]
            torch.cuda.synchronize()
            torch.cuda._sleep(20_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            assert pool.migrate(src, free, s.cuda_stream) == ellm.OK
            e1.record(s)
            torch.cuda.synchronize()
            best = max(best, 2 * n_move * pool.chunk_bytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
        out["bulk" if bulk == "1" else "warp"] = round(best, 1)
    pool.close()
    return out


if __name__ == "__main__":
    c2 = W.c2()
    c2.batch = 1
    res = {"c2_2MiB_x1024": run(c2, 1024), "c4_10MiB_rot_x256": run(W.c4(batch=1), 256)}
    print(json.dumps(res))

"""World-size-2 gloo test of the N>1 host path (CPU): head partition, identical chunk tables
on every shard (deterministic allocation), and the head gather reassembling [B, Hq, d]."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_15155_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_15155_b200 import ellm
        Hq, Hkv, d, L = 32, 8, 128, 32
        kv0, kv1, q0, q1 = shard.head_partition(Hq, Hkv, world, rank)
        T = shard.shard_tokens_per_chunk(16, world)
        pool = ellm.Pool(ellm.DEVICE_NONE, L, q1 - q0, kv1 - kv0, d, T, 512, 400, 8, 64, 32)
        assert pool.chunk_bytes == 2 << 20
        rng = np.random.default_rng(0)  # same op sequence on every rank
        for _ in range(50):
            reqs = rng.choice(8, size=3, replace=False)
            pool.reserve(reqs, rng.integers(0, 200, size=3))
            if rng.integers(0, 3) == 0:
                used = [c for r in range(8) for c in pool.table(r)[0].tolist() if c >= 0]
                if used:
                    pool.deflate(used[:2])
            if rng.integers(0, 5) == 0:
                pool.release(int(rng.integers(0, 8)))
        tabs = np.concatenate([np.r_[pool.table(r)[0], -99, pool.table(r)[1]] for r in range(8)])
        t = torch.from_numpy(tabs.astype(np.int64))
        allt = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        same_tables = all(torch.equal(allt[0], x) for x in allt)
        # gather of head-sharded outputs
        ref = torch.arange(4 * Hq * d, dtype=torch.float32).reshape(4, Hq, d)
        full = shard.gather_heads(ref[:, q0:q1].contiguous(), world)
        q.put((rank, same_tables, bool(torch.equal(full, ref)), (kv0, kv1, q0, q1)))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] for r in res), "chunk tables differ between shards"
    assert all(r[2] for r in res), "head gather mismatch"
    assert res[0][3] == (0, 4, 0, 16) and res[1][3] == (4, 8, 16, 32)


def test_partition_errors():
    with pytest.raises(ValueError):
        shard.head_partition(32, 8, 3, 0)
    assert [shard.head_partition(64, 8, 8, r)[2:] for r in (0, 7)] == [(0, 8), (56, 64)]

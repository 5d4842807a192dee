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
        # a10 setup: IPC handles of every rank's gather window, exchanged in rank order
        hs = shard.exchange_handles(bytes([rank + 1]) * 64, world)
        ok_handles = hs == [bytes([i + 1]) * 64 for i in range(world)]
        q.put((rank, same_tables, bool(torch.equal(full, ref)), (kv0, kv1, q0, q1), ok_handles))
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
    assert all(r[4] for r in res), "IPC handle exchange out of rank order"


def test_partition_errors():
    with pytest.raises(ValueError):
        shard.head_partition(32, 8, 3, 0)
    assert [shard.head_partition(64, 8, 8, r)[2:] for r in (0, 7)] == [(0, 8), (56, 64)]


def test_gather_attach_validation_host_only():
    """a10 (include/ellm.h gather_attach / attention_gather / gather_wait): argument checks run
    before any device work; a host-only pool then reports NO_DEVICE."""
    from paper_2506_15155_b200 import ellm
    L, Hq_loc, Hkv_loc, d, B = 2, 16, 4, 128, 4
    pool = ellm.Pool(ellm.DEVICE_NONE, L, Hq_loc, Hkv_loc, d, 32, 64, 64, B, 16, 0)
    nbytes = shard.gather_window_bytes(L, B, 2 * Hq_loc, d)
    assert nbytes == 4096 + L * B * 32 * d * 2
    wins = [1 << 20, 2 << 20]
    assert pool.attention_gather(0, [0], 0, 0, 1.0) == ellm.INVALID_ARG   # not attached
    assert pool.gather_wait(0) == ellm.INVALID_ARG
    assert pool.gather_wait_next(0) == ellm.INVALID_ARG
    try:  # a handle that cannot be opened (here: no device at all) is a peer failure
        ellm.ipc_open(bytes(ellm.IPC_HANDLE_BYTES))
        raise AssertionError("ipc_open of a null handle succeeded")
    except ellm.EllmError as e:
        assert e.rc == ellm.PEER, e
    assert pool.gather_wait_next(L) == ellm.OUT_OF_RANGE
    assert pool.gather_attach(0, 0, Hq_loc, wins, nbytes) == ellm.OUT_OF_RANGE
    assert pool.gather_attach(9, 0, 9 * Hq_loc, wins * 5, nbytes) == ellm.OUT_OF_RANGE
    assert pool.gather_attach(2, 2, 2 * Hq_loc, wins, nbytes) == ellm.OUT_OF_RANGE
    assert pool.gather_attach(2, 1, 3 * Hq_loc, wins, nbytes) == ellm.INVALID_ARG   # heads
    assert pool.gather_attach(2, 1, 2 * Hq_loc, [1 << 20, 17], nbytes) == ellm.INVALID_ARG  # align
    assert pool.gather_attach(2, 1, 2 * Hq_loc, wins, 4096) == ellm.INVALID_ARG
    assert pool.gather_attach(2, 1, 2 * Hq_loc, wins, nbytes) == ellm.NO_DEVICE
    assert shard.layer_stride(3, 5, 64) == 1920 and shard.layer_stride(1, 1, 4) == 16

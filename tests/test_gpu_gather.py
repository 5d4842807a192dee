"""a10: the head-sharded output gather fused into the attention
epilogue over peer memory (include/ellm.h ellm_attention_gather / ellm_gather_wait).

Only one GPU is available here, so the N ranks run on the same device:
  - in one process: N shard pools, N windows, every pool attached to all N windows — exercises
    the kernel's row placement, the flag accounting and the wait for N = 2, 4, 8;
  - in two processes (gloo for the handle exchange): windows mapped with cudaIpcOpenMemHandle,
    i.e. the same path bench.py takes across GPUs, minus the NVLink hop.
Gathered rows must equal the unsharded fp64 oracle (tolerance, R8), be identical in
every rank's window, and be bit-identical to each shard's own non-gather attention output."""
import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _shards(world, L, Hq, Hkv, d, B, ctx, T, seed):
    from inputs.workload import Workload
    return [Workload("gather", L, Hq, Hkv, d, B, ctx, seed, tokens_per_chunk=T * world, world=world, rank=i,
                     decode_headroom=64) for i in range(world)]


def _read_window(addr, nbytes):
    import torch
    from paper_2506_15155_b200 import ellm
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    assert ellm.memcpy_async(h.data_ptr(), addr, nbytes, torch.cuda.current_stream()) == ellm.OK
    torch.cuda.synchronize()
    return h.numpy().copy()


def _oracle_check(wl_full, rows, samples, step_len, what):
    """rows: uint16 [L, B, Hq, d] gathered output; compare sampled (r, l) with the oracle."""
    import oracle
    from inputs import workload as W
    from tests.twin import check_attention
    scale = 1.0 / np.sqrt(wl_full.head_dim)
    for r, l in samples:
        kk, vv = W.host_kv(wl_full, r, l, step_len)
        ref = oracle.attention_contig(W.host_q(wl_full, r, l), kk, vv, scale)
        check_attention(rows[l, r][None], ref[None], f"{what} r={r} l={l}")


@pytest.mark.parametrize("fold", [False, True], ids=["wait_kernel", "folded_wait"])
@pytest.mark.parametrize("world,shape", [
    (2, (2, 4, 2, 64, 5, 300, 16)),        # C1-like geometry, ragged lengths via ctx 300
    (2, (3, 32, 8, 128, 6, 2000, 16)),     # LLaMA-3-8B heads
    (4, (2, 32, 8, 128, 3, 700, 16)),
    (8, (3, 64, 8, 128, 4, 1500, 32)),     # LLaMA-70B heads, one kv-head per rank
])
def test_gather_in_process(world, shape, fold):
    """fold: layer l's wait is folded into layer l+1's attention launch (gather_wait_next, with
    launch overlap on), only the last layer's wait is a kernel — bench.py's N>1 sequence."""
    import torch
    from paper_2506_15155_b200 import ellm, shard
    from inputs import workload as W
    from inputs.workload import Workload
    L, Hq, Hkv, d, B, ctx, T = shape
    wls = _shards(world, L, Hq, Hkv, d, B, ctx, T, seed=7)
    pools = [W.make_pool(w, 0) for w in wls]
    wins = []
    try:
        for p, w in zip(pools, wls):
            W.prefill(p, w)
        nbytes = shard.gather_window_bytes(L, B, Hq, d)
        stride = shard.layer_stride(B, Hq, d)
        wins = [ellm.gather_window_create(0, nbytes)[0] for _ in range(world)]
        for i, p in enumerate(pools):
            assert p.gather_attach(world, i, Hq, wins, nbytes) == ellm.OK
            if fold:
                assert p.set_launch_overlap(True) == ellm.OK
        reqs, ones = list(range(B)), [1] * B
        scale = 1.0 / np.sqrt(d)
        lens = np.full(B, ctx, np.int64)
        for step in range(2):
            ins = [W.decode_inputs(w, step, lens + step) for w in wls]
            for p in pools:
                assert p.reserve(reqs, ones) == ellm.OK
            for l in range(L):
                for i, p in enumerate(pools):
                    q, k, v = ins[i]
                    if fold and l > 0:
                        assert p.gather_wait_next(l - 1) == ellm.OK
                    assert p.attention_gather(l, reqs, q[l], l * stride, scale, k[l], v[l]) == ellm.OK
                if not fold or l == L - 1:
                    for p in pools:
                        assert p.gather_wait(l) == ellm.OK
        torch.cuda.synchronize()
        data = [_read_window(w, nbytes)[ellm.GATHER_DATA_OFFSET:] for w in wins]
        for i in range(1, world):
            assert np.array_equal(data[0], data[i]), f"window of rank {i} differs from rank 0"
        rows = np.stack([data[0][l * stride: l * stride + B * Hq * d * 2].view(np.uint16).reshape(B, Hq, d)
                         for l in range(L)])
        # bit-identical to each shard's own attention (same plan, same merge order)
        hq = Hq // world
        for i, p in enumerate(pools):
            q = ins[i][0]
            for l in range(L):
                out = torch.empty((B, hq, d), dtype=torch.bfloat16, device="cuda")
                assert p.attention(l, reqs, q[l], out, scale) == ellm.OK
                got = W.np_bits(out)
                assert np.array_equal(got, rows[l][:, i * hq:(i + 1) * hq]), f"rank {i} layer {l}"
        # plain (non-append) attention_gather of the same step rewrites the same bits
        for l in range(L):
            for i, p in enumerate(pools):
                assert p.attention_gather(l, reqs, ins[i][0][l], l * stride, scale) == ellm.OK
            for p in pools:
                assert p.gather_wait(l) == ellm.OK
        torch.cuda.synchronize()
        again = _read_window(wins[-1], nbytes)[ellm.GATHER_DATA_OFFSET:]
        assert np.array_equal(again, data[0])
        full = Workload("gather", L, Hq, Hkv, d, B, ctx, 7, tokens_per_chunk=T, decode_headroom=64)
        _oracle_check(full, rows, [(0, 0), (B - 1, L - 1), (B // 2, 1)], ctx + 2, f"world {world}")
    finally:
        for p in pools:
            p.gather_detach()
            p.close()
        for w in wins:
            ellm.gather_window_destroy(w)
        torch.cuda.synchronize()


def test_gather_errors_on_device():
    import torch
    from paper_2506_15155_b200 import ellm, shard
    from inputs import workload as W
    wls = _shards(2, 1, 4, 2, 64, 2, 40, 16, seed=1)
    pool = W.make_pool(wls[0], 0)
    try:
        W.prefill(pool, wls[0])
        nbytes = shard.gather_window_bytes(1, 2, 4, 64)
        wins = [ellm.gather_window_create(0, nbytes)[0] for _ in range(2)]
        assert pool.gather_attach(2, 0, 4, wins, nbytes) == ellm.OK
        q = torch.zeros((2, 2, 64), dtype=torch.bfloat16, device="cuda")
        assert pool.attention_gather(0, [0, 1], q, 8, 1.0) == ellm.INVALID_ARG          # misaligned
        assert pool.attention_gather(0, [0, 1], q, 16, 1.0) == ellm.OUT_OF_RANGE        # past window
        assert pool.attention_gather(1, [0, 1], q, 0, 1.0) == ellm.OUT_OF_RANGE         # layer
        assert pool.attention_gather(0, [0, 1], q, 0, 1.0, q, q) == ellm.INVALID_ARG    # no reservation
        assert pool.gather_wait(3) == ellm.OUT_OF_RANGE
        assert pool.gather_detach() == ellm.OK
        for w in wins:
            assert ellm.gather_window_destroy(w) == ellm.OK
    finally:
        pool.close()


_TIMEOUT_SCRIPT = textwrap.dedent("""
    import sys, torch
    sys.path.insert(0, {root!r})
    from paper_2506_15155_b200 import ellm, shard
    from inputs import workload as W
    from inputs.workload import Workload
    wl = Workload("g", 1, 4, 2, 64, 2, 40, 1, tokens_per_chunk=32, world=2, rank=0)
    pool = W.make_pool(wl, 0)
    W.prefill(pool, wl)
    nbytes = shard.gather_window_bytes(1, 2, 4, 64)
    wins = [ellm.gather_window_create(0, nbytes)[0] for _ in range(2)]
    assert pool.gather_attach(2, 0, 4, wins, nbytes) == 0
    q = torch.zeros((2, 2, 64), dtype=torch.bfloat16, device="cuda")
    assert pool.attention_gather(0, [0, 1], q, 0, 0.125) == 0
    assert pool.gather_wait(0) == 0     # rank 1 never runs: the wait must time out and trap
    try:
        torch.cuda.synchronize()
    except Exception as e:
        print("TRAPPED", type(e).__name__)
        sys.exit(3)
    print("NO ERROR")
""")


@pytest.mark.parametrize("folded", [False, True])
def test_gather_wait_times_out_instead_of_hanging(folded):
    env = dict(os.environ, ELLM_GATHER_TIMEOUT_MS="300")
    script = _TIMEOUT_SCRIPT.format(root=ROOT)
    if folded:  # the wait rides in the next attention launch's producer instead of a wait kernel
        script = script.replace("assert pool.gather_wait(0) == 0",
                                "assert pool.gather_wait_next(0) == 0\n"
                                "assert pool.attention_gather(0, [0, 1], q, 0, 0.125) == 0")
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 3 and "TRAPPED" in r.stdout, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2506_15155_b200 import ellm, shard
    from inputs import workload as W
    L, Hq, Hkv, d, B, ctx, T = 2, 32, 8, 128, 4, 1200, 16
    wl = _shards(world, L, Hq, Hkv, d, B, ctx, T, seed=9)[rank]
    pool = W.make_pool(wl, 0)
    W.prefill(pool, wl)
    g = shard.PeerGather(pool, world, rank, Hq, L, B, d, device=0)
    reqs, ones = list(range(B)), [1] * B
    scale = 1.0 / np.sqrt(d)
    lens = np.full(B, ctx, np.int64)
    dist.barrier()  # every rank attached before any rank writes
    for step in range(3):
        q, k, v = W.decode_inputs(wl, step, lens + step)
        assert pool.reserve(reqs, ones) == ellm.OK
        for l in range(L):  # bench.py's sequence: waits folded into the next launch, then a kernel
            if l > 0:
                assert pool.gather_wait_next(l - 1) == ellm.OK
            assert pool.attention_gather(l, reqs, q[l], g.offset(l), scale, k[l], v[l]) == ellm.OK
        assert pool.gather_wait(L - 1) == ellm.OK
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, f"win{rank}.npy"), _read_window(g.own, g.nbytes)[ellm.GATHER_DATA_OFFSET:])
    dist.barrier()  # nobody unmaps / frees while a peer may still write
    g.close()
    pool.close()
    dist.destroy_process_group()


def test_gather_two_processes_over_ipc(tmp_path):
    import torch.multiprocessing as mp
    from paper_2506_15155_b200 import shard
    from inputs.workload import Workload
    world = 2
    mp.start_processes(_ipc_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    w0, w1 = (np.load(tmp_path / f"win{i}.npy") for i in range(world))
    assert np.array_equal(w0, w1)
    L, Hq, Hkv, d, B, ctx, T = 2, 32, 8, 128, 4, 1200, 16
    stride = shard.layer_stride(B, Hq, d)
    rows = np.stack([w0[l * stride: l * stride + B * Hq * d * 2].view(np.uint16).reshape(B, Hq, d)
                     for l in range(L)])
    full = Workload("gather", L, Hq, Hkv, d, B, ctx, 9, tokens_per_chunk=T, decode_headroom=64)
    _oracle_check(full, rows, [(0, 0), (3, 1), (2, 0)], ctx + 3, "ipc")

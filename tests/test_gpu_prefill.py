"""f4 — chunked-prefill attention over chunk-mapped KV on tcgen05 (P:871,
P:109-112): the kernel's bf16 output vs the fp64 oracle (O12), within DESIGN.md R8's tolerance,
over ragged query counts (1 .. several 128-key tiles), GQA groups 1/4/8, d = 64/128, chunk
sizes below, equal to and above the 128-key tile, and a two-chunk prefill where the second
chunk attends to the first."""
import numpy as np
import pytest

from tests.twin import Twin

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300, method="thread")]

SHAPES = [  # L, Hq, Hkv, d, T
    (1, 32, 8, 128, 16),
    (1, 8, 1, 128, 16),
    (1, 8, 8, 128, 32),
    (1, 16, 4, 64, 16),
    (1, 8, 2, 128, 256),
    (2, 4, 2, 128, 128),
]


@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_prefill_ragged(shape):
    L, Hq, Hkv, d, T = shape
    rng = np.random.default_rng(sum(shape))
    lens = [300, 17, 1000, 129, 1]
    n_q = [300, 17, 200, 1, 1]
    chunks = sum((n + T - 1) // T for n in lens)
    t = Twin(L, Hq, Hkv, d, T, chunks + 8, chunks + 8, len(lens), (max(lens) + T - 1) // T + 1, 0,
             seed=31, needle=False)
    reqs = list(range(len(lens)))
    assert t.reserve(reqs, lens) == 0
    t.append_all_layers(reqs, lens)
    for l in range(L):
        t.prefill(l, reqs, n_q, rng)
    t.prefill(L - 1, [2, 0], [1000, 5], rng)     # full prefill from position 0 + a short tail


def test_two_chunk_prefill_sees_the_first_chunk():
    rng = np.random.default_rng(5)
    t = Twin(1, 32, 8, 128, 16, 200, 200, 2, 120, 0, seed=3, needle=False)
    assert t.reserve([0, 1], [700, 90]) == 0
    t.append_all_layers([0, 1], [700, 90])
    t.prefill(0, [0, 1], [700, 90], rng)
    assert t.reserve([0, 1], [512, 77]) == 0     # second chunk
    t.append_all_layers([0, 1], [512, 77])
    t.prefill(0, [1, 0], [77, 512], rng)
    t.check_bytes()


def test_prefill_errors_match_oracle():
    rng = np.random.default_rng(9)
    t = Twin(1, 8, 2, 128, 16, 40, 40, 3, 20, 8, seed=2, needle=False)
    assert t.reserve([0, 1], [100, 20]) == 0
    t.append_all_layers([0, 1], [100, 20])
    assert t.prefill(0, [0], [101], rng) == -1   # n_q > len
    assert t.prefill(0, [2], [1], rng) == -1     # empty request
    rc, _ = t.deflate([t.o.table(1)[0][0]])
    assert rc == 0
    assert t.prefill(0, [0, 1], [4, 4], rng) == -5
    t.prefill(0, [0], [100], rng)


def test_prefill_fragmented_tables():
    """Chunk ids of a request in runs of 1..9 (two requests reserving alternately): the producer
    splits each 128-key tile into boxes of 1/2/4/8 consecutive chunks."""
    rng = np.random.default_rng(12)
    t = Twin(1, 32, 8, 128, 16, 400, 400, 2, 200, 0, seed=8, needle=False)
    for _ in range(30):
        for r in (0, 1):
            n = 16 * int(rng.integers(1, 10)) - int(rng.integers(0, 3))
            if t.reserve([r], [n]) == 0:
                t.append_all_layers([r], [n])
    runs = np.diff(t.o.table(0)[0]) == 1
    assert runs.any() and not runs.all()
    lens = [int(t.lens[0]), int(t.lens[1])]
    t.prefill(0, [0, 1], [lens[0], min(lens[1], 333)], rng)

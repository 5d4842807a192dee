"""CPU oracle for the eLLM KV-traffic hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product package
(``paper_2506_15155_b200``) never imports it and shares no code with it.

The oracle is ``oracle/oracle.cpp`` (C++17, fp64, no CUDA) loaded through ctypes,
plus ``oracle/brute.py`` (numpy textbook attention) that pins its arithmetic.
Paper: arXiv 2506.15155 (``/root/reference/PAPER.md``, cited as P:<line>).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

OK, INVALID_ARG, OUT_OF_RANGE, NO_CHUNKS, HOST_FULL, NOT_RESIDENT, NOT_MAPPED, ALREADY_MAPPED, IN_USE = (
    0, -1, -2, -3, -4, -5, -6, -7, -8)


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (-fopenmp). Building the checker is not using it."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
                               "-Wall", "-o", _SO, _SRC])
    return _SO


class _Cfg(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("n_heads_q", ctypes.c_int32),
                ("n_heads_kv", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("tokens_per_chunk", ctypes.c_int32), ("max_chunks", ctypes.c_int64),
                ("initial_chunks", ctypes.c_int64), ("max_requests", ctypes.c_int32),
                ("max_chunks_per_request", ctypes.c_int32), ("host_slots", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        _lib.eo_create.restype = P
        _lib.eo_create.argtypes = [ctypes.POINTER(_Cfg)]
        _lib.eo_destroy.argtypes = [P]
        _lib.eo_chunk_bytes.restype = I64
        _lib.eo_chunk_bytes.argtypes = [P]
        for name, args in {
            "eo_reserve": [P, I32, P, P],
            "eo_append": [P, I32, I32, P, P, P, P],
            "eo_attention": [P, I32, I32, P, P, ctypes.c_double, P, I32],
            "eo_prefill_attention": [P, I32, I32, P, P, P, ctypes.c_double, P, I32],
            "eo_deflate": [P, I32, P, P],
            "eo_inflate": [P, I32, P, P],
            "eo_migrate": [P, I32, P, P],
            "eo_release": [P, I32],
            "eo_grow": [P, I64],
            "eo_shrink": [P, I64],
            "eo_act_alloc": [P, I64, P],
            "eo_act_free": [P, I64],
            "eo_stats": [P, P],
            "eo_get_table": [P, I32, P, I32, P, P],
            "eo_read_chunk": [P, I64, P],
            "eo_read_host_slot": [P, I64, P],
            "eo_check_invariants": [P],
            "eo_attention_contig": [I32, I32, I32, I32, P, P, P, ctypes.c_double, P],
            "eo_num_threads": [],
        }.items():
            f = getattr(_lib, name)
            f.restype = ctypes.c_int
            f.argtypes = args
        _lib.eo_act_used.restype = I64
        _lib.eo_act_used.argtypes = [P]
    return _lib


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def attention_contig(q_bits: np.ndarray, k_bits: np.ndarray, v_bits: np.ndarray,
                     scale: float) -> np.ndarray:
    """Stateless fp64 textbook attention for one request/layer.

    q_bits [Hq, d] uint16 (bf16 bits); k_bits, v_bits [len, Hkv, d] uint16. Returns [Hq, d] f64.
    """
    q = np.ascontiguousarray(q_bits, dtype=np.uint16)
    k = np.ascontiguousarray(k_bits, dtype=np.uint16)
    v = np.ascontiguousarray(v_bits, dtype=np.uint16)
    Hq, d = q.shape
    n, Hkv, d2 = k.shape
    assert d2 == d and v.shape == k.shape
    out = np.empty((Hq, d), dtype=np.float64)
    rc = lib().eo_attention_contig(Hq, Hkv, d, n, _ptr(q), _ptr(k), _ptr(v), float(scale), _ptr(out))
    if rc != OK:
        raise ValueError(f"eo_attention_contig rc={rc}")
    return out


def num_threads() -> int:
    return int(lib().eo_num_threads())


class Oracle:
    """Stateful oracle pool. Methods return (rc, outputs...)."""

    def __init__(self, n_layers, n_heads_q, n_heads_kv, head_dim, tokens_per_chunk, max_chunks,
                 initial_chunks, max_requests, max_chunks_per_request, host_slots):
        self.cfg = dict(n_layers=n_layers, n_heads_q=n_heads_q, n_heads_kv=n_heads_kv,
                        head_dim=head_dim, tokens_per_chunk=tokens_per_chunk,
                        max_chunks=max_chunks, initial_chunks=initial_chunks,
                        max_requests=max_requests, max_chunks_per_request=max_chunks_per_request,
                        host_slots=host_slots)
        c = _Cfg(**self.cfg)
        self._h = lib().eo_create(ctypes.byref(c))
        if not self._h:
            raise ValueError("bad oracle config")
        self.chunk_bytes = int(lib().eo_chunk_bytes(self._h))

    def close(self):
        if self._h:
            lib().eo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reserve(self, reqs, n_new):
        r, n = _i32(reqs), _i32(n_new)
        return lib().eo_reserve(self._h, len(r), _ptr(r), _ptr(n))

    def append(self, layer, reqs, n_new, k_bits, v_bits):
        r, n = _i32(reqs), _i32(n_new)
        k = np.ascontiguousarray(k_bits, dtype=np.uint16)
        v = np.ascontiguousarray(v_bits, dtype=np.uint16)
        return lib().eo_append(self._h, layer, len(r), _ptr(r), _ptr(n), _ptr(k), _ptr(v))

    def attention(self, layer, reqs, q_bits, scale, through_table=True):
        r = _i32(reqs)
        q = np.ascontiguousarray(q_bits, dtype=np.uint16)
        out = np.zeros((len(r), self.cfg["n_heads_q"], self.cfg["head_dim"]), dtype=np.float64)
        rc = lib().eo_attention(self._h, layer, len(r), _ptr(r), _ptr(q), float(scale), _ptr(out),
                                1 if through_table else 0)
        return rc, out

    def prefill_attention(self, layer, reqs, n_q, q_bits, scale, through_table=True):
        """O12 (f4): causal attention of the last n_q[i] positions of each request."""
        r, nq = _i32(reqs), _i32(n_q)
        q = np.ascontiguousarray(q_bits, dtype=np.uint16)
        rows = int(nq.sum()) if len(nq) else 0
        out = np.zeros((rows, self.cfg["n_heads_q"], self.cfg["head_dim"]), dtype=np.float64)
        rc = lib().eo_prefill_attention(self._h, layer, len(r), _ptr(r), _ptr(nq), _ptr(q), float(scale),
                                        _ptr(out), 1 if through_table else 0)
        return rc, out

    def deflate(self, ids):
        a = _i32(ids)
        out = np.full(len(a), -1, dtype=np.int32)
        rc = lib().eo_deflate(self._h, len(a), _ptr(a), _ptr(out))
        return rc, out

    def inflate(self, slots):
        a = _i32(slots)
        out = np.full(len(a), -1, dtype=np.int32)
        rc = lib().eo_inflate(self._h, len(a), _ptr(a), _ptr(out))
        return rc, out

    def migrate(self, src, dst):
        s, d = _i32(src), _i32(dst)
        if len(s) != len(d):
            return INVALID_ARG
        return lib().eo_migrate(self._h, len(s), _ptr(s), _ptr(d))

    def release(self, req):
        return lib().eo_release(self._h, int(req))

    def grow(self, n):
        return lib().eo_grow(self._h, int(n))

    def shrink(self, n):
        return lib().eo_shrink(self._h, int(n))

    def act_alloc(self, n_chunks):
        """O10 (f3): returns (rc, first chunk of the activation slot)."""
        first = ctypes.c_int64(-1)
        rc = lib().eo_act_alloc(self._h, int(n_chunks), ctypes.byref(first))
        return rc, first.value

    def act_free(self, first):
        """O11 (f3)."""
        return lib().eo_act_free(self._h, int(first))

    def stats(self):
        out = np.zeros(5, dtype=np.int64)
        lib().eo_stats(self._h, _ptr(out))
        d = dict(zip(("kv_free", "kv_used", "act", "host_free", "host_used"), out.tolist()))
        d["act_used"] = int(lib().eo_act_used(self._h))
        return d

    def table(self, req):
        cap = self.cfg["max_chunks_per_request"]
        ent = np.full(cap, -1, dtype=np.int32)
        n = ctypes.c_int32(0)
        ln = ctypes.c_int32(0)
        rc = lib().eo_get_table(self._h, int(req), _ptr(ent), cap, ctypes.byref(n), ctypes.byref(ln))
        if rc != OK:
            raise ValueError(f"eo_get_table rc={rc}")
        return ent[: n.value].copy(), ln.value

    def read_chunk(self, c):
        buf = np.zeros(self.chunk_bytes, dtype=np.uint8)
        rc = lib().eo_read_chunk(self._h, int(c), _ptr(buf))
        if rc != OK:
            raise ValueError(f"eo_read_chunk rc={rc}")
        return buf

    def read_host_slot(self, h):
        buf = np.zeros(self.chunk_bytes, dtype=np.uint8)
        rc = lib().eo_read_host_slot(self._h, int(h), _ptr(buf))
        if rc != OK:
            raise ValueError(f"eo_read_host_slot rc={rc}")
        return buf

    def check_invariants(self):
        return int(lib().eo_check_invariants(self._h))

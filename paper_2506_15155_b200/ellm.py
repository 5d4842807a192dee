"""Thin ctypes binding of libellm.so (include/ellm.h) — argument marshalling only.

Every step of the hot path runs in libellm.so's CUDA kernels; there is no CPU fallback:
importing this module raises if the library is missing. Function names match the C ABI.
Tensors are passed as device pointers (``tensor.data_ptr()``); host metadata as Python
sequences / numpy arrays; streams as ``torch.cuda.Stream.cuda_stream`` integers (0 = default).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ELLM_LIB_PATH: another in-tree build of the same sources (A/B measurements of build variants)
LIB_PATH = os.environ.get("ELLM_LIB_PATH") or os.path.join(_HERE, "libellm.so")

OK = 0
ERR = {
    -1: "INVALID_ARG", -2: "OUT_OF_RANGE", -3: "NO_CHUNKS", -4: "HOST_FULL", -5: "NOT_RESIDENT",
    -6: "NOT_MAPPED", -7: "ALREADY_MAPPED", -8: "IN_USE", -9: "CUDA", -10: "PEER", -11: "NO_DEVICE",
    -12: "UNSUPPORTED",
}
(INVALID_ARG, OUT_OF_RANGE, NO_CHUNKS, HOST_FULL, NOT_RESIDENT, NOT_MAPPED, ALREADY_MAPPED, IN_USE,
 CUDA, PEER, NO_DEVICE, UNSUPPORTED) = range(-1, -13, -1)
DEVICE_NONE = -1

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2506_15155_b200.build` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)


class ellm_pool_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("n_layers", ctypes.c_int32), ("n_heads_q", ctypes.c_int32),
                ("n_heads_kv", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("tokens_per_chunk", ctypes.c_int32), ("max_chunks", ctypes.c_int64),
                ("initial_chunks", ctypes.c_int64), ("max_requests", ctypes.c_int32),
                ("max_chunks_per_request", ctypes.c_int32), ("host_slots", ctypes.c_int64),
                ("map_unit_bytes", ctypes.c_int64)]


class ellm_stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("kv_free", "kv_used", "act", "host_free", "host_used", "n_map",
                                               "n_unmap", "map_ns", "unmap_ns", "chunk_bytes", "mapped_bytes",
                                               "premapped_bytes", "pending_unmap", "crit_vmm_ns",
                                               "n_steal", "premap_hits", "act_used", "act_cached_bytes")]


_P, _V = ctypes.c_void_p, ctypes.c_void_p
_I32, _I64 = ctypes.c_int32, ctypes.c_int64
_SIGS = {
    "ellm_vmm_granularity": (ctypes.c_int, [_I32, ctypes.POINTER(ctypes.c_size_t)]),
    "ellm_vtensor_create": (ctypes.c_int, [_I32, ctypes.c_size_t, _I64, ctypes.POINTER(_P)]),
    "ellm_vtensor_map": (ctypes.c_int, [_P, _I64, _I64]),
    "ellm_vtensor_unmap": (ctypes.c_int, [_P, _I64, _I64]),
    "ellm_vtensor_is_mapped": (ctypes.c_int, [_P, _I64]),
    "ellm_vtensor_base": (_V, [_P]),
    "ellm_vtensor_destroy": (ctypes.c_int, [_P]),
    "ellm_pool_create": (ctypes.c_int, [ctypes.POINTER(ellm_pool_config), ctypes.POINTER(_P)]),
    "ellm_pool_destroy": (ctypes.c_int, [_P]),
    "ellm_pool_stats": (ctypes.c_int, [_P, ctypes.POINTER(ellm_stats)]),
    "ellm_pool_base": (_V, [_P]),
    "ellm_pool_host_base": (_V, [_P]),
    "ellm_kv_reserve": (ctypes.c_int, [_P, _I32, _P, _P, _V]),
    "ellm_kv_append": (ctypes.c_int, [_P, _I32, _I32, _P, _P, _V, _V, _V]),
    "ellm_paged_decode_attention": (ctypes.c_int, [_P, _I32, _I32, _P, _V, _V, ctypes.c_float, _V]),
    "ellm_decode_append_attention": (ctypes.c_int, [_P, _I32, _I32, _P, _V, _V, _V, _V, ctypes.c_float, _V]),
    "ellm_release": (ctypes.c_int, [_P, _I32, _V]),
    "ellm_deflate": (ctypes.c_int, [_P, _I32, _P, _P, _V]),
    "ellm_inflate": (ctypes.c_int, [_P, _I32, _P, _P, _V]),
    "ellm_migrate": (ctypes.c_int, [_P, _I32, _P, _P, _V]),
    "ellm_offload_begin": (ctypes.c_int, [_P, _I32, _P, _P]),
    "ellm_offload_layer": (ctypes.c_int, [_P, _I32, _I32, _P, _V]),
    "ellm_offload_commit": (ctypes.c_int, [_P, _I32, _P, _V]),
    "ellm_pool_grow": (ctypes.c_int, [_P, _I64]),
    "ellm_pool_shrink": (ctypes.c_int, [_P, _I64]),
    "ellm_set_swap_mode": (ctypes.c_int, [_P, _I32]),
    "ellm_set_vmm_overlap": (ctypes.c_int, [_P, ctypes.c_int64, _I32]),
    "ellm_set_launch_overlap": (ctypes.c_int, [_P, _I32]),
    "ellm_vmm_sync": (ctypes.c_int, [_P]),
    "ellm_prefill_attention": (ctypes.c_int, [_P, _I32, _I32, _P, _P, _P, _P, ctypes.c_float, _P]),
    "ellm_act_alloc": (ctypes.c_int, [_P, ctypes.c_int64, _P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_P)]),
    "ellm_act_free": (ctypes.c_int, [_P, ctypes.c_int64, _P]),
    "ellm_act_trim": (ctypes.c_int, [_P]),
    "ellm_torch_set_pool": (ctypes.c_int, [_P]),
    "ellm_torch_alloc": (_P, [ctypes.c_size_t, ctypes.c_int, _P]),
    "ellm_torch_free": (None, [_P, ctypes.c_size_t, ctypes.c_int, _P]),
    "ellm_get_table": (ctypes.c_int, [_P, _I32, _P, _I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "ellm_chunk_states": (ctypes.c_int, [_P, _I64, _I64, _P]),
    "ellm_read_chunk": (ctypes.c_int, [_P, _I64, _V, _V]),
    "ellm_read_host_slot": (ctypes.c_int, [_P, _I64, _V]),
    "ellm_alias_request": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_V)]),
    "ellm_unalias_request": (ctypes.c_int, [_P, _I32]),
    "ellm_gather_window_create": (ctypes.c_int, [_I32, _I64, ctypes.POINTER(_V), _P]),
    "ellm_gather_window_destroy": (ctypes.c_int, [_V]),
    "ellm_ipc_open": (ctypes.c_int, [_P, ctypes.POINTER(_V)]),
    "ellm_ipc_close": (ctypes.c_int, [_V]),
    "ellm_gather_attach": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _I64]),
    "ellm_gather_detach": (ctypes.c_int, [_P]),
    "ellm_attention_gather": (ctypes.c_int, [_P, _I32, _I32, _P, _V, _V, _V, _I64, ctypes.c_float, _V]),
    "ellm_gather_wait": (ctypes.c_int, [_P, _I32, _V]),
    "ellm_gather_wait_next": (ctypes.c_int, [_P, _I32]),
    "ellm_set_attn_trace": (ctypes.c_int, [_P, _V, _I32]),
    "ellm_debug_attn_weights": (ctypes.c_int, [_P, _P, _I32]),
    "ellm_memcpy_async": (ctypes.c_int, [_V, _V, _I64, _V]),
    "ellm_upload": (ctypes.c_int, [_P, _V, _V, _I64, _V]),
    "ellm_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "ellm_last_cuda_error": (ctypes.c_int, [_P]),
    "ellm_kernel_launches": (_I64, [_P]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f

EXPORTS = tuple(_SIGS)


class EllmError(RuntimeError):
    def __init__(self, rc: int, what: str):
        super().__init__(f"{what}: {ERR.get(rc, rc)} ({rc})")
        self.rc = rc


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dptr(t) -> int:
    """Device pointer of a torch tensor (or an int address)."""
    return t if isinstance(t, int) else t.data_ptr()


def _sptr(stream) -> int:
    if stream is None:
        return 0
    return stream if isinstance(stream, int) else stream.cuda_stream


class Pool:
    """Owning wrapper around an ``ellm_pool*``. Methods return the C status code (0 = OK)
    unless noted; ``check=True`` raises EllmError on a non-zero code instead."""

    def __init__(self, device: int, n_layers: int, n_heads_q: int, n_heads_kv: int, head_dim: int,
                 tokens_per_chunk: int, max_chunks: int, initial_chunks: int, max_requests: int,
                 max_chunks_per_request: int, host_slots: int = 0, map_unit_bytes: int = 0):
        self.cfg = ellm_pool_config(device, n_layers, n_heads_q, n_heads_kv, head_dim, tokens_per_chunk,
                                    max_chunks, initial_chunks, max_requests, max_chunks_per_request,
                                    host_slots, map_unit_bytes)
        h = _P()
        rc = ellm_pool_create(ctypes.byref(self.cfg), ctypes.byref(h))
        if rc != OK:
            raise EllmError(rc, "ellm_pool_create")
        self._h = h
        self.chunk_bytes = self.stats()["chunk_bytes"]

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            ellm_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> dict:
        s = ellm_stats()
        rc = ellm_pool_stats(self._h, ctypes.byref(s))
        if rc != OK:
            raise EllmError(rc, "ellm_pool_stats")
        return {n: getattr(s, n) for n, _ in ellm_stats._fields_}

    def base(self) -> int:
        return ellm_pool_base(self._h) or 0

    def reserve(self, reqs, n_new, stream=None) -> int:
        r, n = _i32(reqs), _i32(n_new)
        return ellm_kv_reserve(self._h, len(r), _ptr(r), _ptr(n), _sptr(stream))

    def append(self, layer, reqs, n_new, k_new, v_new, stream=None) -> int:
        r, n = _i32(reqs), _i32(n_new)
        return ellm_kv_append(self._h, layer, len(r), _ptr(r), _ptr(n), _dptr(k_new), _dptr(v_new),
                              _sptr(stream))

    def attention(self, layer, reqs, q, out, scale, stream=None) -> int:
        r = _i32(reqs)
        return ellm_paged_decode_attention(self._h, layer, len(r), _ptr(r), _dptr(q), _dptr(out),
                                           float(scale), _sptr(stream))

    def decode_append_attention(self, layer, reqs, k_new, v_new, q, out, scale, stream=None) -> int:
        """kv_append of one token per request + attention, fused in one launch."""
        r = _i32(reqs)
        return ellm_decode_append_attention(self._h, layer, len(r), _ptr(r), _dptr(k_new), _dptr(v_new),
                                            _dptr(q), _dptr(out), float(scale), _sptr(stream))

    # ---- a10: head-sharded output gather fused into the attention epilogue (peer memory) ----
    def gather_attach(self, world: int, rank: int, heads_q_total: int, windows, window_bytes: int) -> int:
        """windows[i]: device address of rank i's gather window in this process."""
        arr = (_V * len(windows))(*[int(w) for w in windows])
        return ellm_gather_attach(self._h, int(world), int(rank), int(heads_q_total), ctypes.cast(arr, _P),
                                  int(window_bytes))

    def gather_detach(self) -> int:
        return ellm_gather_detach(self._h)

    def attention_gather(self, layer, reqs, q, out_offset, scale, k_new=None, v_new=None, stream=None) -> int:
        """Attention (fused with the decode append when k_new / v_new are given) whose
        [n, Hq_total, d] output rows land in every rank's window at out_offset."""
        r = _i32(reqs)
        return ellm_attention_gather(self._h, int(layer), len(r), _ptr(r),
                                     _dptr(k_new) if k_new is not None else None,
                                     _dptr(v_new) if v_new is not None else None, _dptr(q), int(out_offset),
                                     float(scale), _sptr(stream))

    def gather_wait(self, layer, stream=None) -> int:
        return ellm_gather_wait(self._h, int(layer), _sptr(stream))

    def debug_attn_weights(self, w) -> int:
        """Static split weights per attention CTA (measurement knob); [] restores equal shares."""
        a = np.ascontiguousarray(np.asarray(w, dtype=np.float32))
        return ellm_debug_attn_weights(self._h, a.ctypes.data_as(ctypes.c_void_p) if a.size else None, int(a.size))

    def set_attn_trace(self, device_buf, launches: int) -> int:
        """Per-CTA timeline stamps of the next attention launches (profiling)."""
        return ellm_set_attn_trace(self._h, _dptr(device_buf) if device_buf is not None else None, int(launches))

    def gather_wait_next(self, layer) -> int:
        """Fold the wait for `layer`'s gather into this pool's next attention launch."""
        return ellm_gather_wait_next(self._h, int(layer))

    def release(self, req, stream=None) -> int:
        return ellm_release(self._h, int(req), _sptr(stream))

    def deflate(self, ids, stream=None):
        a = _i32(ids)
        out = np.full(len(a), -1, np.int32)
        rc = ellm_deflate(self._h, len(a), _ptr(a), _ptr(out), _sptr(stream))
        return rc, out

    def inflate(self, slots, stream=None):
        a = _i32(slots)
        out = np.full(len(a), -1, np.int32)
        rc = ellm_inflate(self._h, len(a), _ptr(a), _ptr(out), _sptr(stream))
        return rc, out

    def offload_begin(self, ids):
        a = _i32(ids)
        out = np.full(len(a), -1, np.int32)
        rc = ellm_offload_begin(self._h, len(a), _ptr(a), _ptr(out))
        return rc, out

    def offload_layer(self, layer, ids, stream=None) -> int:
        a = _i32(ids)
        return ellm_offload_layer(self._h, int(layer), len(a), _ptr(a), _sptr(stream))

    def offload_commit(self, ids, stream=None) -> int:
        a = _i32(ids)
        return ellm_offload_commit(self._h, len(a), _ptr(a), _sptr(stream))

    def migrate(self, src, dst, stream=None) -> int:
        s, d = _i32(src), _i32(dst)
        if len(s) != len(d):
            return INVALID_ARG
        return ellm_migrate(self._h, len(s), _ptr(s), _ptr(d), _sptr(stream))

    def grow(self, n) -> int:
        return ellm_pool_grow(self._h, int(n))

    def shrink(self, n) -> int:
        return ellm_pool_shrink(self._h, int(n))

    def set_swap_mode(self, mode: int) -> int:
        return ellm_set_swap_mode(self._h, int(mode))

    def upload(self, dst, src, nbytes=None, stream=None) -> int:
        """host -> device copy staged through the pool's side-context buffer (ellm_upload);
        dst: device tensor or pointer, src: pinned host tensor or pointer."""
        if nbytes is None:
            nbytes = src.numel() * src.element_size()
        return ellm_upload(self._h, _dptr(dst), _dptr(src), int(nbytes), _sptr(stream))

    def set_vmm_overlap(self, premap_bytes: int = 0, async_unmap: bool = False) -> int:
        """f1: speculative pre-mapping budget and asynchronous unmapping."""
        return ellm_set_vmm_overlap(self._h, int(premap_bytes), int(bool(async_unmap)))

    def set_launch_overlap(self, enable: bool = True) -> int:
        """PDL between back-to-back attention launches of this pool (off by default)."""
        return ellm_set_launch_overlap(self._h, int(bool(enable)))

    def vmm_sync(self) -> int:
        return ellm_vmm_sync(self._h)

    def prefill_attention(self, layer, reqs, n_q, q, out, scale, stream=None) -> int:
        """f4: causal attention of the last n_q[i] positions of each request (tcgen05)."""
        r, nq = _i32(reqs), _i32(n_q)
        return ellm_prefill_attention(self._h, int(layer), len(r), _ptr(r), _ptr(nq), _dptr(q), _dptr(out),
                                      float(scale), _sptr(stream))

    # ---- f3: activation eTensors in the unified pool ----
    def act_alloc(self, nbytes_or_chunks, stream=None, chunks=True):
        """Activation slot; returns (rc, first chunk). `chunks=True`: the size is in chunks."""
        nbytes = int(nbytes_or_chunks) * self.chunk_bytes if chunks else int(nbytes_or_chunks)
        first = ctypes.c_int64(-1)
        ptr = _P()
        rc = ellm_act_alloc(self._h, nbytes, _sptr(stream), ctypes.byref(first), ctypes.byref(ptr))
        self._last_act_ptr = ptr.value
        return rc, first.value

    def act_free(self, first, stream=None) -> int:
        return ellm_act_free(self._h, int(first), _sptr(stream))

    def act_trim(self) -> int:
        return ellm_act_trim(self._h)

    def activation_mempool(self):
        """A torch.cuda.MemPool whose segments are activation slots of this pool (torch's
        caching allocator keeps its best-fit/coalescing strategy on top). Use with
        torch.cuda.use_mem_pool(mp). One pool at a time is registered for the hooks."""
        import torch
        ellm_torch_set_pool(self._h)
        alloc = torch.cuda.memory.CUDAPluggableAllocator(LIB_PATH, "ellm_torch_alloc", "ellm_torch_free")
        return torch.cuda.MemPool(alloc.allocator())

    def table(self, req):
        cap = self.cfg.max_chunks_per_request
        ent = np.full(cap, -1, np.int32)
        n, ln = _I32(0), _I32(0)
        rc = ellm_get_table(self._h, int(req), _ptr(ent), cap, ctypes.byref(n), ctypes.byref(ln))
        if rc != OK:
            raise EllmError(rc, "ellm_get_table")
        return ent[: n.value].copy(), ln.value

    def chunk_states(self) -> np.ndarray:
        """uint8 [max_chunks]: 0 FREE, 1 USED, 2 ACT (idle), 3 ACT inside a live activation slot."""
        out = np.zeros(self.cfg.max_chunks, np.uint8)
        rc = ellm_chunk_states(self._h, 0, self.cfg.max_chunks, _ptr(out))
        if rc != OK:
            raise EllmError(rc, "ellm_chunk_states")
        return out

    def free_chunks(self) -> list[int]:
        """FREE KV chunk ids, ascending."""
        return np.flatnonzero(self.chunk_states() == 0).tolist()

    def read_chunk(self, c, stream=None) -> np.ndarray:
        buf = np.zeros(self.chunk_bytes, np.uint8)
        rc = ellm_read_chunk(self._h, int(c), _ptr(buf), _sptr(stream))
        if rc != OK:
            raise EllmError(rc, "ellm_read_chunk")
        return buf

    def read_host_slot(self, h) -> np.ndarray:
        buf = np.zeros(self.chunk_bytes, np.uint8)
        rc = ellm_read_host_slot(self._h, int(h), _ptr(buf))
        if rc != OK:
            raise EllmError(rc, "ellm_read_host_slot")
        return buf

    def alias_request(self, req) -> tuple[int, int]:
        p = _V()
        rc = ellm_alias_request(self._h, int(req), ctypes.byref(p))
        return rc, (p.value or 0)

    def unalias_request(self, req) -> int:
        return ellm_unalias_request(self._h, int(req))

    def last_cuda_error(self) -> int:
        return ellm_last_cuda_error(self._h)

    def kernel_launches(self) -> int:
        return int(ellm_kernel_launches(self._h))


def status_string(rc: int) -> str:
    return ellm_status_string(rc).decode()


def vmm_granularity(device: int = 0) -> int:
    g = ctypes.c_size_t(0)
    rc = ellm_vmm_granularity(device, ctypes.byref(g))
    if rc != OK:
        raise EllmError(rc, "ellm_vmm_granularity")
    return g.value


GATHER_DATA_OFFSET = 4096  # include/ellm.h ELLM_GATHER_DATA_OFFSET
IPC_HANDLE_BYTES = 64


def gather_window_create(device: int, nbytes: int) -> tuple[int, bytes]:
    """(device address, 64-byte cudaIpcMemHandle) of a fresh zeroed gather window."""
    w = _V()
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    rc = ellm_gather_window_create(int(device), int(nbytes), ctypes.byref(w), ctypes.cast(h, _P))
    if rc != OK:
        raise EllmError(rc, "ellm_gather_window_create")
    return w.value, h.raw


def gather_window_destroy(addr: int) -> int:
    return ellm_gather_window_destroy(addr)


def ipc_open(handle: bytes) -> int:
    w = _V()
    buf = ctypes.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES)
    rc = ellm_ipc_open(ctypes.cast(buf, _P), ctypes.byref(w))
    if rc != OK:
        raise EllmError(rc, "ellm_ipc_open")
    return w.value


def ipc_close(addr: int) -> int:
    return ellm_ipc_close(addr)


def memcpy_async(dst, src, nbytes: int, stream=None) -> int:
    """cudaMemcpyAsync(cudaMemcpyDefault) between raw addresses / tensors (window readback)."""
    return ellm_memcpy_async(_dptr(dst), _dptr(src), int(nbytes), _sptr(stream))

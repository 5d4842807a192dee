// pool.cpp — host side of libellm.so: chunk pool with KV/ACT ownership, per-request
// chunk tables (the KV eTensor's logical->physical map), pinned host slots (the CPU
// elastic buffer), and the C-ABI entry points of include/ellm.h that drive the
// kernels in kernels.cu / attention.cu.
//
// Every entry point validates all preconditions before mutating (include/ellm.h
// "Conventions"); allocation is lowest-id-first (R7).
#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <set>

#include "internal.h"

using namespace ellm;

namespace {

constexpr int32_t UNMAPPED = -1;
inline bool is_dev(int32_t e) { return e >= 0; }
inline bool is_host(int32_t e) { return e <= -2; }
inline int32_t host_of(int32_t e) { return -e - 2; }
inline int32_t enc_host(int64_t h) { return int32_t(-(h + 2)); }
constexpr uint8_t KV = 0, ACT = 1;

int cuda_fail(ellm_pool* p, cudaError_t e) {
  if (p) p->last_cuda_error = int(e);
  return ELLM_ERR_CUDA;
}

bool has_dup(int32_t n, const int32_t* a) {
  if (n <= 1) return false;
  std::vector<int32_t> v(a, a + n);
  std::sort(v.begin(), v.end());
  return std::adjacent_find(v.begin(), v.end()) != v.end();
}

int64_t nchunks_of(const ellm_pool* p, int64_t len) { return (len + p->T - 1) / p->T; }
int32_t& entry(ellm_pool* p, int32_t r, int64_t i) {
  return p->table[size_t(int64_t(r) * p->cfg.max_chunks_per_request + i)];
}
int32_t entry_c(const ellm_pool* p, int32_t r, int64_t i) {
  return p->table[size_t(int64_t(r) * p->cfg.max_chunks_per_request + i)];
}
void set_entry(ellm_pool* p, int32_t r, int64_t i, int32_t v) {
  entry(p, r, i) = v;
  ++p->table_epoch;  // invalidates host-built attention descriptors (dynamic-unit entries)
  p->pending_updates.push_back(
      {int32_t(int64_t(r) * p->cfg.max_chunks_per_request + i), v});
}

int64_t take_lowest_free_kv(ellm_pool* p) {
  for (int64_t c = p->free_hint; c < p->cfg.max_chunks; ++c)
    if (p->owner[size_t(c)] == KV && !p->used[size_t(c)]) {
      p->used[size_t(c)] = 1;
      p->free_hint = c + 1;
      --p->n_free_kv;
      ++p->n_used_kv;
      return c;
    }
  return -1;
}
void free_chunk(ellm_pool* p, int64_t c) {
  p->used[size_t(c)] = 0;
  p->chunk_req[size_t(c)] = -1;
  ++p->n_free_kv;
  --p->n_used_kv;
  p->free_hint = std::min(p->free_hint, c);
}
int64_t take_lowest_free_host(ellm_pool* p) {
  for (int64_t h = p->host_hint; h < p->cfg.host_slots; ++h)
    if (!p->hused[size_t(h)]) {
      p->hused[size_t(h)] = 1;
      p->host_hint = h + 1;
      ++p->n_host_used;
      return h;
    }
  return -1;
}
void free_host(ellm_pool* p, int64_t h) {
  p->hused[size_t(h)] = 0;
  p->slot_req[size_t(h)] = -1;
  --p->n_host_used;
  p->host_hint = std::min(p->host_hint, h);
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Copy-engine (DMA) copies. Each piece is (dst, src, bytes); pieces are issued as one
// cudaMemcpyAsync per maximal contiguous run (both sides advance by the piece size) or one
// cudaMemcpy2DAsync per maximal strided run (equal sizes, constant dst and src strides: e.g.
// consecutive chunk ids whose host slots are consecutive, or one layer slab of each). The host
// cost is then per run, not per chunk; the copies are exact byte copies either way.
struct CopyPiece {
  uint8_t* d;
  const uint8_t* s;
  int64_t n;
};
// ELLM_CE_MAX_COPY (bytes, measurement knob; 0 = unlimited): split contiguous runs into copies of
// at most this size (C3 swap-in interference study).
static int64_t ce_max_copy() {
  static const int64_t v = [] {
    const char* e = std::getenv("ELLM_CE_MAX_COPY");
    return e ? std::max<int64_t>(0, std::atoll(e)) : int64_t(0);
  }();
  return v;
}
cudaError_t issue_copies(const std::vector<CopyPiece>& pc, cudaStream_t stream) {
  const int64_t cap = ce_max_copy();
  size_t i = 0;
  while (i < pc.size()) {
    const CopyPiece& a = pc[i];
    size_t j = i + 1;
    if (j < pc.size() && pc[j].n == a.n && pc[j].d - a.d >= a.n && pc[j].s - a.s >= a.n) {
      const int64_t dp = pc[j].d - a.d, sp = pc[j].s - a.s;
      while (j < pc.size() && pc[j].n == a.n && pc[j].d - pc[j - 1].d == dp && pc[j].s - pc[j - 1].s == sp) ++j;
      const size_t rows = j - i;
      cudaError_t e;
      if (dp == a.n && sp == a.n) {
        const int64_t total = a.n * int64_t(rows);
        const int64_t step = cap > 0 ? std::max<int64_t>(a.n, cap / a.n * a.n) : total;
        e = cudaSuccess;
        for (int64_t off = 0; off < total && e == cudaSuccess; off += step)
          e = cudaMemcpyAsync(a.d + off, a.s + off, size_t(std::min(step, total - off)), cudaMemcpyDefault, stream);
      } else {
        // strided run: rows of a.n bytes, split into groups of at most `cap` bytes as well
        const size_t step = cap > 0 ? std::max<size_t>(1, size_t(cap / a.n)) : rows;
        e = cudaSuccess;
        for (size_t r0 = 0; r0 < rows && e == cudaSuccess; r0 += step)
          e = cudaMemcpy2DAsync(a.d + int64_t(r0) * dp, size_t(dp), a.s + int64_t(r0) * sp, size_t(sp), size_t(a.n),
                                std::min(step, rows - r0), cudaMemcpyDefault, stream);
      }
      if (e != cudaSuccess) return e;
    } else {
      cudaError_t e = cudaMemcpyAsync(a.d, a.s, size_t(a.n), cudaMemcpyDefault, stream);
      if (e != cudaSuccess) return e;
    }
    i = j;
  }
  return cudaSuccess;
}

// Copy-engine path of deflate / inflate: dst_base[dst[i]] <- src_base[src[i]], chunk_bytes each.
// With rotated slabs (rot = L) the pool side of chunk c holds canonical layers [0, L-r) at slots
// [r, L) and [L-r, L) at [0, r), r = slab_shift(c): two pieces per chunk (dev_side: 1 = src,
// 2 = dst). The pieces are listed piece-major (all first pieces, then all second pieces) so that
// chunks of one rotation group with consecutive ids and slots form one strided run each.
cudaError_t ce_copy(uint8_t* dst_base, const std::vector<int32_t>& dst, const uint8_t* src_base,
                    const std::vector<int32_t>& src, int64_t chunk_bytes, cudaStream_t stream,
                    int32_t rot = 0, int64_t slab = 0, int dev_side = 0) {
  std::vector<CopyPiece> pc;
  pc.reserve(dst.size());
  for (int k = 0; k < 2; ++k)
    for (size_t i = 0; i < dst.size(); ++i) {
      uint8_t* dc = dst_base + int64_t(dst[i]) * chunk_bytes;
      const uint8_t* sc = src_base + int64_t(src[i]) * chunk_bytes;
      const int64_t r = slab_shift(dev_side == 1 ? src[i] : dst[i], rot);
      if (r == 0) {
        if (k == 0) pc.push_back({dc, sc, chunk_bytes});
        continue;
      }
      // canonical layers [0, L-r) <-> device slots [r, L); layers [L-r, L) <-> slots [0, r)
      const int64_t canon_off = k == 0 ? 0 : (rot - r) * slab, dev_off = k == 0 ? r * slab : 0;
      const int64_t len = k == 0 ? (rot - r) * slab : r * slab;
      if (dev_side == 1)
        pc.push_back({dc + canon_off, sc + dev_off, len});
      else
        pc.push_back({dc + dev_off, sc + canon_off, len});
    }
  return issue_copies(pc, stream);
}

// Swap mode 3 and ellm_upload: host -> device copies staged through memory owned by a second CUDA
// context on the pool's device. Measured (tools/interference_ctx2.py, DESIGN.md §5 C3): a
// concurrent 128 GiB decode step slows 2.33x while host -> device copies land in memory allocated
// by the decode's own context, 1.67x when another context issues them into that memory, but only
// 1.06-1.09x when they land in memory allocated by another context — and 1.09-1.11x when the data
// then moves on into the decode's memory by device -> device copies, issued from either context.
// So the second context exists only to own a 256 MiB staging buffer; every copy is issued on the
// caller's stream from the caller's context: host -> staging (copy engine, one copy per run),
// then staging -> destination (device -> device). The staging buffer is reused in stream order;
// a use on another stream first waits for the previous use (side_ev). Driver failures creating
// the context are reported as ELLM_ERR_CUDA with last_cuda_error = 10000 + CUresult.
constexpr int64_t kSideStageBytes = int64_t(256) << 20;
void side_destroy(ellm_pool* p);
int side_init(ellm_pool* p) {
  if (p->side_ctx) return ELLM_OK;
  const CtxDriver& d = ctx_driver();
  if (!d.ok) return ELLM_ERR_UNSUPPORTED;
  CUdevice dev;
  CUcontext c = nullptr, prev = nullptr;
  CUresult r = d.deviceGet(&dev, p->cfg.device);
  if (r == CUDA_SUCCESS) r = d.ctxCreate(&c, 0, dev);
  if (r != CUDA_SUCCESS) {
    p->last_cuda_error = 10000 + int(r);
    return ELLM_ERR_CUDA;
  }
  // cuCtxCreate made `c` current: the staging buffer is allocated by (owned by) that context
  const int64_t stage = std::max<int64_t>(1, kSideStageBytes / p->chunk_bytes) * p->chunk_bytes;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p->side_stage), size_t(stage));
  d.ctxPopCurrent(&prev);
  p->side_ctx = c;
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->side_ev, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    const int rc = cuda_fail(p, e);
    side_destroy(p);
    return rc;
  }
  p->side_stage_bytes = stage;
  p->side_ev_used = false;
  return ELLM_OK;
}
void side_destroy(ellm_pool* p) {
  if (!p->side_ctx) return;
  const CtxDriver& d = ctx_driver();
  if (d.ctxPushCurrent(p->side_ctx) == CUDA_SUCCESS) {
    if (p->side_stage) cudaFree(p->side_stage);
    CUcontext prev;
    d.ctxPopCurrent(&prev);
  }
  if (p->side_ev) cudaEventDestroy(p->side_ev);
  d.ctxDestroy(p->side_ctx);
  p->side_ctx = nullptr;
  p->side_ev = nullptr;
  p->side_stage = nullptr;
}
// before `stream` reuses the staging buffer: wait for its previous use on another stream
cudaError_t side_acquire(ellm_pool* p, cudaStream_t stream) {
  if (p->side_ev_used && p->side_ev_stream != stream) return cudaStreamWaitEvent(stream, p->side_ev, 0);
  return cudaSuccess;
}
cudaError_t side_release(ellm_pool* p, cudaStream_t stream) {
  p->side_ev_stream = stream;
  p->side_ev_used = true;
  return cudaEventRecord(p->side_ev, stream);
}
// pool chunks dst[i] <- host slots src[i] through the staging buffer, on `stream`
cudaError_t side_inflate_copy(ellm_pool* p, uint8_t* pool, const std::vector<int32_t>& dst,
                              const std::vector<int32_t>& src, cudaStream_t stream) {
  cudaError_t e = side_acquire(p, stream);
  const int64_t S_chunks = p->side_stage_bytes / p->chunk_bytes;
  for (size_t b0 = 0; b0 < dst.size() && e == cudaSuccess; b0 += size_t(S_chunks)) {
    const size_t k = std::min(dst.size() - b0, size_t(S_chunks));
    std::vector<int32_t> sidx(k), hs(src.begin() + int64_t(b0), src.begin() + int64_t(b0 + k)),
        ds(dst.begin() + int64_t(b0), dst.begin() + int64_t(b0 + k));
    for (size_t i = 0; i < k; ++i) sidx[i] = int32_t(i);
    e = ce_copy(p->side_stage, sidx, p->host_slots, hs, p->chunk_bytes, stream);  // host link
    if (e == cudaSuccess)  // canonical staging image -> (rotated) chunk slabs
      e = ce_copy(pool, ds, p->side_stage, sidx, p->chunk_bytes, stream, p->ash.rot, p->ash.slab, 2);
  }
  if (e == cudaSuccess) e = side_release(p, stream);
  return e;
}

// ---- stream-ordered reuse of freed chunks / host slots (see ellm_pool::FreeEvent) ----------
// Record an event on `stream` after the work that frees some chunks / slots; returns its index.
int32_t record_free_event(ellm_pool* p, cudaStream_t stream) {
  int32_t i;
  if (!p->free_event_pool.empty()) {
    i = p->free_event_pool.back();
    p->free_event_pool.pop_back();
  } else {
    ellm_pool::FreeEvent fe;
    if (cudaEventCreateWithFlags(&fe.ev, cudaEventDisableTiming) != cudaSuccess) return -1;
    p->free_events.push_back(fe);
    i = int32_t(p->free_events.size()) - 1;
  }
  ellm_pool::FreeEvent& fe = p->free_events[size_t(i)];
  fe.stream = stream;
  fe.refs = 0;
  if (cudaEventRecord(fe.ev, stream) != cudaSuccess) return -1;
  return i;
}
void drop_ref(ellm_pool* p, int32_t i) {
  if (i >= 0 && --p->free_events[size_t(i)].refs == 0) p->free_event_pool.push_back(i);
}
void attach_event(ellm_pool* p, std::vector<int32_t>& tag, int64_t id, int32_t i) {
  drop_ref(p, tag[size_t(id)]);
  tag[size_t(id)] = i;
  if (i >= 0) ++p->free_events[size_t(i)].refs;
}
// Before work on `stream` touches a newly allocated chunk / slot: wait for its freeing work
// if that ran on another stream.
cudaError_t wait_freed(ellm_pool* p, std::vector<int32_t>& tag, int64_t id, cudaStream_t stream) {
  const int32_t i = tag[size_t(id)];
  if (i < 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  if (p->free_events[size_t(i)].stream != stream) {
    static const bool dbg = std::getenv("ELLM_DEBUG_WAITS") != nullptr;  // measurement aid
    if (dbg && cudaEventQuery(p->free_events[size_t(i)].ev) == cudaErrorNotReady)
      std::fprintf(stderr, "[ellm] stream %p waits for unfinished work on stream %p (%s %lld)\n",
                   static_cast<void*>(stream), static_cast<void*>(p->free_events[size_t(i)].stream),
                   &tag == &p->chunk_ev ? "chunk" : "slot", static_cast<long long>(id));
    e = cudaStreamWaitEvent(stream, p->free_events[size_t(i)].ev, 0);
  }
  tag[size_t(id)] = -1;
  drop_ref(p, i);
  return e;
}

// Upload pending table updates (snapshots of host entries) and scatter them on `stream`.
int flush_table(ellm_pool* p, cudaStream_t stream) {
  if (!p->has_dev) {
    p->pending_updates.clear();
    return ELLM_OK;
  }
  const size_t per = p->ring.seg_bytes() / sizeof(TableUpdate);
  size_t done = 0;
  while (done < p->pending_updates.size()) {
    size_t n = std::min(per, p->pending_updates.size() - done);
    void *h, *d;
    int rc = p->ring.alloc(n * sizeof(TableUpdate), &h, &d, nullptr);
    if (rc) return rc;
    std::memcpy(h, p->pending_updates.data() + done, n * sizeof(TableUpdate));
    if ((rc = p->ring.upload(d, n * sizeof(TableUpdate), stream))) return rc;
    cudaError_t e = launch_table_scatter(p->d_table, static_cast<TableUpdate*>(d), int32_t(n), stream);
    if (e != cudaSuccess) return cuda_fail(p, e);
    ++p->launches;
    if ((rc = p->ring.commit(stream))) return rc;
    done += n;
  }
  p->pending_updates.clear();
  return ELLM_OK;
}

// Upload an int32 array through the staging ring; returns the device pointer.
// Grid of the SM copy kernels that move chunks over the host link (deflate, inflate, layer-wise
// offload): one CTA per SM — the room the persistent decode-attention kernel leaves beside it —
// which already keeps ~4.7 MB of PCIe traffic in flight (measured 51.9 GB/s, the same as with
// 2 CTAs per SM). ELLM_HOST_COPY_CTAS overrides (experiments).
int host_copy_grid(const ellm_pool* p) {
  static const int env = [] {
    const char* e = std::getenv("ELLM_HOST_COPY_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  return env > 0 ? env : p->num_sms;
}

int upload_ints(ellm_pool* p, const std::vector<int32_t>& v, cudaStream_t stream,
                const int32_t** dev, uint64_t* gen) {
  void *h, *d;
  int rc = p->ring.alloc(std::max<size_t>(v.size(), 1) * 4, &h, &d, gen);
  if (rc) return rc;
  if (!v.empty()) std::memcpy(h, v.data(), v.size() * 4);
  if ((rc = p->ring.upload(d, std::max<size_t>(v.size(), 1) * 4, stream))) return rc;
  *dev = static_cast<const int32_t*>(d);
  return ELLM_OK;
}

// ---- f1: VMM overlap (see ellm_pool) — the *_units helpers run with vmm_mu held -----------
// Units that should be mapped: every unit holding a KV chunk, plus the premap window (the
// premap_units lowest all-ACT units: pool_grow takes the lowest ACT ids next).
inline bool unit_live(const ellm_pool* p, size_t u) {  // must stay mapped regardless of policy
  return p->unit_kv[u] > 0 || p->unit_act[u] > 0 || p->act_cached[u];
}
std::vector<uint8_t> wanted_units(const ellm_pool* p) {
  std::vector<uint8_t> w(p->unit_kv.size(), 0);
  int64_t k = 0;
  for (size_t u = 0; u < w.size(); ++u)
    if (unit_live(p, u)) w[u] = 1;
    else if (k < p->premap_units) w[u] = 1, ++k;
  return w;
}

// Make every unit in `need` (sorted) mapped with its own memory, on the caller's thread (vmm_mu
// held). A unit still mapped but "doomed" is unmapped first; with async unmapping on, a unit
// awaiting its unmap (mapped, not live, outside the premap window, not in `keep`) donates its
// physical handle instead of a fresh cuMemCreate (multi-mapping).
int map_units_now(ellm_pool* p, const std::set<int64_t>& need, const std::set<int64_t>& keep) {
  bool synced = false;
  std::vector<int64_t> fresh;
  for (int64_t u : need) {
    if (p->vt->mapped[size_t(u)] && !p->doomed[size_t(u)]) continue;
    if (p->doomed[size_t(u)]) {  // its old VA mapping must go before it is reused
      if (!synced && cudaDeviceSynchronize() != cudaSuccess) return ELLM_ERR_CUDA;
      synced = true;
      if (int rc = vt_unmap_slot_nosync(p->vt, u)) return rc;
      p->doomed[size_t(u)] = 0;
    }
    int64_t donor = -1;
    if (p->async_unmap) {
      const std::vector<uint8_t> want = wanted_units(p);
      for (int64_t v = int64_t(p->unit_kv.size()) - 1; v >= 0 && donor < 0; --v)
        if (p->vt->mapped[size_t(v)] && !p->doomed[size_t(v)] && !unit_live(p, size_t(v)) &&
            !want[size_t(v)] && !keep.count(v) && !need.count(v))
          donor = v;
    }
    if (donor >= 0) {
      if (int rc = vt_map_from(p->vt, u, donor)) return rc;
      p->doomed[size_t(donor)] = 1;
      ++p->n_steal;
      // the memory's pending users are those of the donor's chunks: carry their free events
      for (int64_t k = 0; k < p->chunks_per_unit; ++k) {
        const int64_t cu = u * p->chunks_per_unit + k, cv = donor * p->chunks_per_unit + k;
        if (cu < p->cfg.max_chunks && cv < p->cfg.max_chunks)
          attach_event(p, p->chunk_ev, cu, p->chunk_ev[size_t(cv)]);
      }
    } else {
      fresh.push_back(u);
    }
  }
  for (size_t i = 0; i < fresh.size();) {  // map contiguous runs at once
    size_t k = i + 1;
    while (k < fresh.size() && fresh[k] == fresh[k - 1] + 1) ++k;
    if (int rc = ellm_vtensor_map(p->vt, fresh[i], int64_t(k - i))) return rc;
    i = k;
  }
  return ELLM_OK;
}

// Synchronous release (async unmapping off): unmap the given units that are no longer wanted.
int unmap_units_now(ellm_pool* p, std::vector<int64_t> units) {
  const std::vector<uint8_t> want = wanted_units(p);
  std::sort(units.begin(), units.end());
  bool synced = false;
  for (int64_t u : units)
    if (!want[size_t(u)] && p->vt->mapped[size_t(u)]) {
      if (!synced && cudaDeviceSynchronize() != cudaSuccess) return ELLM_ERR_CUDA;
      synced = true;
      if (int rc = vt_unmap_slot_nosync(p->vt, u)) return rc;
      p->doomed[size_t(u)] = 0;
    }
  return ELLM_OK;
}

void vmm_kick(ellm_pool* p) {  // called with vmm_mu held
  if (!p->vmm_started) return;
  p->vmm_dirty = true;
  p->vmm_cv.notify_all();
}

// Worker: unmap doomed / unwanted units (after a device sync, so work enqueued before their
// chunks became ACT has finished), then map the premap window. Each driver call runs with
// vmm_mu held, so pool_grow / pool_shrink see consistent unit state.
void vmm_worker(ellm_pool* p) {
  cudaSetDevice(p->cfg.device);
  std::unique_lock<std::mutex> lk(p->vmm_mu);
  for (;;) {
    p->vmm_cv.wait(lk, [&] { return p->vmm_stop || p->vmm_dirty; });
    if (p->vmm_stop) break;
    p->vmm_dirty = false;
    p->vmm_busy = true;
    if (p->vmm_delay_us > 0) {
      lk.unlock();
      std::this_thread::sleep_for(std::chrono::microseconds(p->vmm_delay_us));
      lk.lock();
    }
    std::vector<uint8_t> want = wanted_units(p);
    std::vector<std::pair<int64_t, uint64_t>> cand;  // (unit, generation) before the sync
    for (size_t u = 0; u < want.size(); ++u)
      if (p->vt->mapped[u] && !unit_live(p, u) && (p->doomed[u] || !want[u]))
        cand.push_back({int64_t(u), p->unit_gen[u]});
    if (!cand.empty()) {
      lk.unlock();
      const cudaError_t e = cudaDeviceSynchronize();
      lk.lock();
      if (e != cudaSuccess) p->vmm_error = ELLM_ERR_CUDA;
      want = wanted_units(p);
      for (auto [u, gen] : cand) {  // re-check: a grow may have taken the unit back meanwhile
        if (e != cudaSuccess || !p->vt->mapped[size_t(u)] || unit_live(p, size_t(u)) ||
            p->unit_gen[size_t(u)] != gen || !(p->doomed[size_t(u)] || !want[size_t(u)]))
          continue;
        if (vt_unmap_slot_nosync(p->vt, u) != ELLM_OK) p->vmm_error = ELLM_ERR_CUDA;
        p->doomed[size_t(u)] = 0;
      }
    }
    want = wanted_units(p);
    for (size_t u = 0; u < want.size() && !p->vmm_stop; ++u)
      if (want[u] && !p->vt->mapped[u] && ellm_vtensor_map(p->vt, int64_t(u), 1) != ELLM_OK)
        p->vmm_error = ELLM_ERR_CUDA;
    p->vmm_busy = false;
    p->vmm_cv.notify_all();
  }
}

bool check_reqs_range(const ellm_pool* p, int32_t n, const int32_t* r) {
  for (int32_t i = 0; i < n; ++i)
    if (r[i] < 0 || r[i] >= p->cfg.max_requests) return false;
  return true;
}

}  // namespace

extern "C" {

const char* ellm_status_string(int s) {
  switch (s) {
    case ELLM_OK: return "ok";
    case ELLM_ERR_INVALID_ARG: return "invalid argument";
    case ELLM_ERR_OUT_OF_RANGE: return "out of range";
    case ELLM_ERR_NO_CHUNKS: return "not enough free KV chunks";
    case ELLM_ERR_HOST_FULL: return "not enough free host slots";
    case ELLM_ERR_NOT_RESIDENT: return "chunk not resident on the device";
    case ELLM_ERR_NOT_MAPPED: return "chunk or slot not in use / not mapped";
    case ELLM_ERR_ALREADY_MAPPED: return "destination already in use";
    case ELLM_ERR_IN_USE: return "chunks in use";
    case ELLM_ERR_CUDA: return "CUDA error";
    case ELLM_ERR_PEER: return "peer gather window could not be opened";
    case ELLM_ERR_NO_DEVICE: return "pool has no device";
    case ELLM_ERR_UNSUPPORTED: return "unsupported shape";
    default: return "unknown status";
  }
}

int ellm_last_cuda_error(const ellm_pool* p) { return p ? p->last_cuda_error : 0; }
int64_t ellm_kernel_launches(const ellm_pool* p) { return p ? p->launches : 0; }

int ellm_debug_attn_weights(ellm_pool* p, const float* w, int32_t n) {
  if (!p || n < 0 || (n > 0 && !w)) return ELLM_ERR_INVALID_ARG;
  p->dbg_weights.assign(w, w + n);
  p->cache_key.clear();
  return ELLM_OK;
}

int ellm_set_attn_trace(ellm_pool* p, void* device_buf, int32_t launches) {
  if (!p || launches < 0 || (device_buf && launches == 0)) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  p->trace_buf = static_cast<unsigned long long*>(device_buf);
  p->trace_slots = device_buf ? launches : 0;
  p->trace_launch = 0;
  return ELLM_OK;
}

// Split-K state of the attention launches, sized for calls of up to `reqs` list entries
// (duplicates allowed, so a call may list more than max_requests): partial records
// pid < (G + 2 n_vr + n_dyn) * nsub, each [HB*group][D] fp32 + (m, l), and one arrival counter
// per virtual request (zero between launches). Grown on demand by attention_impl; growing
// synchronises the device (in-flight launches use the old buffers).
static int alloc_attn_state(ellm_pool* p, int64_t reqs) {
  const AttnShape& a = p->ash;
  const int64_t group = a.group;
  if (p->d_part || p->d_part_ml || p->d_arrivals) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(p, e);
    cudaFree(p->d_part);
    cudaFree(p->d_part_ml);
    cudaFree(p->d_arrivals);
    p->d_part = p->d_part_ml = nullptr;
    p->d_arrivals = nullptr;
  }
  p->part_records = (int64_t(p->num_sms) + 2 * reqs * a.HG + kMaxDynUnits) * a.nsub;
  cudaError_t e;
  if ((e = cudaMalloc(reinterpret_cast<void**>(&p->d_part),
                      size_t(p->part_records) * a.HB * group * a.D * 4)) != cudaSuccess ||
      (e = cudaMalloc(reinterpret_cast<void**>(&p->d_part_ml),
                      size_t(p->part_records) * a.HB * group * 2 * 4)) != cudaSuccess ||
      (e = cudaMalloc(reinterpret_cast<void**>(&p->d_arrivals), size_t(reqs) * a.HG * 4)) != cudaSuccess ||
      (e = cudaMemset(p->d_arrivals, 0, size_t(reqs) * a.HG * 4)) != cudaSuccess)
    return cuda_fail(p, e);
  p->attn_cap = reqs;
  return ELLM_OK;
}

int ellm_pool_create(const ellm_pool_config* cfg, ellm_pool** out) {
  if (!cfg || !out) return ELLM_ERR_INVALID_ARG;
  *out = nullptr;
  const ellm_pool_config& c = *cfg;
  if (c.n_layers <= 0 || c.n_heads_q <= 0 || c.n_heads_kv <= 0 || c.head_dim <= 0 ||
      c.tokens_per_chunk <= 0 || c.max_chunks <= 0 || c.initial_chunks < 0 ||
      c.initial_chunks > c.max_chunks || c.max_requests <= 0 || c.max_chunks_per_request <= 0 ||
      c.host_slots < 0 || c.n_heads_q % c.n_heads_kv != 0 || c.max_chunks > INT32_MAX ||
      c.host_slots > INT32_MAX - 2 ||
      int64_t(c.max_requests) * c.max_chunks_per_request > INT32_MAX)
    return ELLM_ERR_INVALID_ARG;
  const int32_t T = c.tokens_per_chunk, group = c.n_heads_q / c.n_heads_kv;
  if ((c.head_dim != 64 && c.head_dim != 128) || T < 16 || (T & (T - 1)) != 0 || group > 8 ||
      (c.n_heads_kv & (c.n_heads_kv - 1)) != 0)
    return ELLM_ERR_UNSUPPORTED;

  ellm_pool* p = new ellm_pool();
  p->cfg = c;
  p->T = T;
  p->group = group;
  p->chunk_bytes = int64_t(4) * T * c.n_layers * c.n_heads_kv * c.head_dim;
  p->has_dev = c.device != ELLM_DEVICE_NONE;
  // schedule tuning knobs (defaults documented in DESIGN.md §5)
  if (const char* v = std::getenv("ELLM_ATTN_DYN_DIV")) p->dyn_div = std::max(0L, std::atol(v));
  if (const char* v = std::getenv("ELLM_ATTN_DYN_UNIT")) p->dyn_unit = std::max(1L, std::atol(v));
  p->owner.assign(size_t(c.max_chunks), ACT);
  p->used.assign(size_t(c.max_chunks), 0);
  for (int64_t i = 0; i < c.initial_chunks; ++i) p->owner[size_t(i)] = KV;
  p->n_free_kv = c.initial_chunks;
  p->n_act = c.max_chunks - c.initial_chunks;
  p->chunk_req.assign(size_t(c.max_chunks), -1);
  p->chunk_idx.assign(size_t(c.max_chunks), -1);
  p->hused.assign(size_t(c.host_slots), 0);
  p->slot_req.assign(size_t(c.host_slots), -1);
  p->slot_idx.assign(size_t(c.host_slots), -1);
  p->chunk_ev.assign(size_t(c.max_chunks), -1);
  p->act_len.assign(size_t(c.max_chunks), 0);
  p->in_act.assign(size_t(c.max_chunks), 0);
  p->slot_ev.assign(size_t(c.host_slots), -1);
  p->off_slot.assign(size_t(c.max_chunks), -1);
  p->off_words = (c.n_layers + 63) / 64;
  p->off_layers.assign(size_t(c.max_chunks) * size_t(p->off_words), 0);
  p->table.assign(size_t(int64_t(c.max_requests) * c.max_chunks_per_request), UNMAPPED);
  p->len.assign(size_t(c.max_requests), 0);
  p->pending.assign(size_t(c.max_requests), 0);
  p->nonres.assign(size_t(c.max_requests), 0);
  if (!p->has_dev) {
    *out = p;
    return ELLM_OK;
  }

  auto fail = [&](int rc) {
    ellm_pool_destroy(p);
    return rc;
  };
  cudaError_t e;
  if (c.device < 0 || (e = cudaSetDevice(c.device)) != cudaSuccess) return fail(ELLM_ERR_CUDA);
  if (!driver().ok) return fail(ELLM_ERR_CUDA);
  size_t gran = 0;
  int rc = ellm_vmm_granularity(c.device, &gran);
  if (rc) return fail(rc);
  // Physical map unit: a multiple of lcm(chunk_bytes, granularity). Driver VMM cost on B200 is
  // per handle (cuMemCreate ~0.1 ms, cuMemSetAccess ~0.2-1 ms per handle, measured), so the
  // default unit is >= 64 MiB; KV/ACT ownership stays per chunk and a unit's memory is released
  // once all of its chunks are ACT (R1, §5).
  const int64_t g64 = int64_t(gran);
  int64_t lcm = p->chunk_bytes;
  while (lcm % g64 != 0) lcm += p->chunk_bytes;
  int64_t want_unit = c.map_unit_bytes;
  if (want_unit == 0)
    if (const char* v = std::getenv("ELLM_MAP_UNIT_BYTES")) want_unit = std::atol(v);  // experiments
  if (want_unit > 0) {
    if (want_unit % lcm != 0) return fail(ELLM_ERR_UNSUPPORTED);
    p->unit_bytes = want_unit;
  } else {
    p->unit_bytes = lcm * (((int64_t(64) << 20) + lcm - 1) / lcm);
    const int64_t pool_bytes = ((c.max_chunks * p->chunk_bytes + lcm - 1) / lcm) * lcm;
    p->unit_bytes = std::min(p->unit_bytes, pool_bytes);
  }
  p->chunks_per_unit = p->unit_bytes / p->chunk_bytes;
  int64_t n_units = (c.max_chunks + p->chunks_per_unit - 1) / p->chunks_per_unit;
  if ((rc = ellm_vtensor_create(c.device, size_t(p->unit_bytes), n_units, &p->vt))) return fail(rc);
  p->unit_kv.assign(size_t(n_units), 0);
  p->unit_gen.assign(size_t(n_units), 0);
  p->unit_act.assign(size_t(n_units), 0);
  p->act_cached.assign(size_t(n_units), 0);
  p->doomed.assign(size_t(n_units), 0);
  if (const char* v = std::getenv("ELLM_VMM_WORKER_DELAY_US")) p->vmm_delay_us = std::max(0L, std::atol(v));
  for (int64_t i = 0; i < c.initial_chunks; ++i) ++p->unit_kv[size_t(i / p->chunks_per_unit)];
  for (int64_t u = 0; u < n_units;) {  // map runs of units that hold KV chunks
    int64_t v = u;
    while (v < n_units && p->unit_kv[size_t(v)] > 0) ++v;
    if (v > u && (rc = ellm_vtensor_map(p->vt, u, v - u))) return fail(rc);
    u = v + 1;
  }
  if (c.host_slots > 0) {
    if ((e = cudaHostAlloc(reinterpret_cast<void**>(&p->host_slots),
                           size_t(c.host_slots) * size_t(p->chunk_bytes),
                           cudaHostAllocMapped | cudaHostAllocPortable)) != cudaSuccess)
      return fail(cuda_fail(p, e));
  }
  size_t tbytes = p->table.size() * 4;
  if ((e = cudaMalloc(reinterpret_cast<void**>(&p->d_table), tbytes)) != cudaSuccess ||
      (e = cudaMemset(p->d_table, 0xFF, tbytes)) != cudaSuccess)
    return fail(cuda_fail(p, e));
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, c.device)) != cudaSuccess) return fail(cuda_fail(p, e));
  p->num_sms = prop.multiProcessorCount;

  AttnShape& a = p->ash;
  a.D = c.head_dim;
  a.Hkv = c.n_heads_kv;
  a.Hq = c.n_heads_q;
  a.group = group;
  a.HB = attn_heads_per_block(c.n_heads_kv);
  a.HG = c.n_heads_kv / a.HB;
  a.TT = attn_stage_tokens(a.HB);
  a.nsub = a.TT / 16;
  a.T = T;
  a.L = c.n_layers;
  // rotated slabs (internal.h slab_slot): used when the chunk stride is not a
  // power of two (power-of-two strides read at full rate canonically, and the rotation costs the
  // prefill kernel ~8%), and possible unless a chunk is its own map unit (ellm_alias_request's
  // contiguous per-request view needs the canonical image), the layer count is 1, or a slab is
  // not a whole number of 4 KiB copy units. ELLM_ROTATE=1 / 0 forces it on / off.
  a.slab = p->chunk_bytes / c.n_layers;
  const bool can_rot = c.n_layers > 1 && p->chunks_per_unit > 1 && a.slab % 4096 == 0;
  bool want_rot = (p->chunk_bytes & (p->chunk_bytes - 1)) != 0;
  if (const char* v = std::getenv("ELLM_ROTATE")) want_rot = std::atoi(v) != 0;
  a.rot = (can_rot && want_rot) ? c.n_layers : 0;
  if ((rc = alloc_attn_state(p, c.max_requests))) return fail(rc);
  // d_ticket[0]: dynamic-unit tickets; d_ticket[1] (low word): CTAs finished in gather launches
  if ((e = cudaMalloc(reinterpret_cast<void**>(&p->d_ticket), 16)) != cudaSuccess ||
      (e = cudaMemset(p->d_ticket, 0, 16)) != cudaSuccess)
    return fail(cuda_fail(p, e));
  if ((rc = p->ring.init(size_t(1) << 20, 16))) return fail(rc);
  if ((e = encode_kv_tensor_map(&p->tmap, ellm_vtensor_base(p->vt), c.max_chunks, a)) != cudaSuccess)
    return fail(cuda_fail(p, e));
  if ((e = attn_configure(a.D, a.HB)) != cudaSuccess) return fail(cuda_fail(p, e));
  if (const char* v = std::getenv("ELLM_PDL")) {
    p->pdl = std::atoi(v) != 0;
    p->pdl_env = true;
  }
  *out = p;
  return ELLM_OK;
}

int ellm_pool_destroy(ellm_pool* p) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  if (p->vmm_started) {
    {
      std::lock_guard<std::mutex> g(p->vmm_mu);
      p->vmm_stop = true;
    }
    p->vmm_cv.notify_all();
    p->vmm_thread.join();
  }
  if (p->has_dev) {
    cudaSetDevice(p->cfg.device);
    cudaDeviceSynchronize();
    for (auto it = p->alias.begin(); it != p->alias.end();) {
      int32_t r = it->first;
      ++it;
      ellm_unalias_request(p, r);
    }
    p->ring.destroy();
    for (auto& fe : p->free_events)
      if (fe.ev) cudaEventDestroy(fe.ev);
    if (p->d_table) cudaFree(p->d_table);
    if (p->d_stage) cudaFree(p->d_stage);
    if (p->stage_ev) cudaEventDestroy(p->stage_ev);
    side_destroy(p);
    if (p->d_part) cudaFree(p->d_part);
    if (p->d_part_ml) cudaFree(p->d_part_ml);
    if (p->d_arrivals) cudaFree(p->d_arrivals);
    if (p->d_ticket) cudaFree(p->d_ticket);
    if (p->host_slots) cudaFreeHost(p->host_slots);
    if (p->vt) ellm_vtensor_destroy(p->vt);
  }
  delete p;
  return ELLM_OK;
}

int ellm_pool_stats(const ellm_pool* p, ellm_stats* o) {
  if (!p || !o) return ELLM_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> g(const_cast<ellm_pool*>(p)->vmm_mu);
  o->kv_free = p->n_free_kv;
  o->kv_used = p->n_used_kv;
  o->act = p->n_act;
  o->host_used = p->n_host_used;
  o->host_free = p->cfg.host_slots - p->n_host_used;
  o->n_map = p->vt ? p->vt->n_map : 0;
  o->n_unmap = p->vt ? p->vt->n_unmap : 0;
  o->map_ns = p->vt ? p->vt->map_ns : 0;
  o->unmap_ns = p->vt ? p->vt->unmap_ns : 0;
  o->chunk_bytes = p->chunk_bytes;
  int64_t mapped = 0;
  if (p->vt)
    for (uint8_t m : p->vt->mapped) mapped += m;
  o->mapped_bytes = mapped * p->unit_bytes;
  o->premapped_bytes = o->pending_unmap = 0;
  if (p->vt) {
    const std::vector<uint8_t> want = wanted_units(p);
    for (size_t u = 0; u < want.size(); ++u)
      if (p->vt->mapped[u] && !unit_live(p, u)) {
        if (p->doomed[u] || !want[u]) ++o->pending_unmap;
        else o->premapped_bytes += p->unit_bytes;
      }
  }
  o->act_used = p->n_act_used;
  o->act_cached_bytes = 0;
  for (size_t u = 0; u < p->act_cached.size(); ++u)
    if (p->act_cached[u] && p->unit_act[u] == 0 && p->unit_kv[u] == 0) o->act_cached_bytes += p->unit_bytes;
  o->crit_vmm_ns = p->crit_vmm_ns;
  o->n_steal = p->n_steal;
  o->premap_hits = p->premap_hits;
  return ELLM_OK;
}

void* ellm_pool_base(const ellm_pool* p) { return p && p->vt ? ellm_vtensor_base(p->vt) : nullptr; }
void* ellm_pool_host_base(const ellm_pool* p) { return p ? p->host_slots : nullptr; }

int ellm_set_swap_mode(ellm_pool* p, int32_t mode) {
  if (!p || mode < 0 || mode > 3) return ELLM_ERR_INVALID_ARG;
  if (mode == 3 && p->has_dev) {
    if (cudaSetDevice(p->cfg.device) != cudaSuccess) return ELLM_ERR_CUDA;
    const int rc = side_init(p);
    if (rc) return rc;
  }
  p->swap_mode = mode;
  return ELLM_OK;
}

int ellm_upload(ellm_pool* p, void* dst, const void* src, int64_t bytes, void* stream) {
  if (!p || bytes < 0 || (bytes > 0 && (!dst || !src))) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  if (bytes == 0) return ELLM_OK;
  if (cudaSetDevice(p->cfg.device) != cudaSuccess) return ELLM_ERR_CUDA;
  const int rc = side_init(p);
  if (rc) return rc;
  cudaStream_t st = S(stream);
  cudaError_t e = side_acquire(p, st);
  for (int64_t off = 0; off < bytes && e == cudaSuccess; off += p->side_stage_bytes) {
    const size_t n = size_t(std::min(p->side_stage_bytes, bytes - off));
    e = cudaMemcpyAsync(p->side_stage, static_cast<const uint8_t*>(src) + off, n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, p->side_stage, n, cudaMemcpyDeviceToDevice, st);
  }
  if (e == cudaSuccess) e = side_release(p, st);
  return e == cudaSuccess ? ELLM_OK : cuda_fail(p, e);
}

// a2 — O2 in SURVEY §8(c): on-demand chunk mapping at write, all-or-nothing.
int ellm_kv_reserve(ellm_pool* p, int32_t n, const int32_t* reqs, const int32_t* n_new,
                    void* stream) {
  if (!p || n < 0 || (n > 0 && (!reqs || !n_new))) return ELLM_ERR_INVALID_ARG;
  if (!check_reqs_range(p, n, reqs)) return ELLM_ERR_OUT_OF_RANGE;
  if (has_dup(n, reqs)) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (n_new[i] < 0) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (nchunks_of(p, p->len[size_t(reqs[i])] + n_new[i]) > p->cfg.max_chunks_per_request)
      return ELLM_ERR_OUT_OF_RANGE;
  for (int32_t i = 0; i < n; ++i) {
    int64_t L = p->len[size_t(reqs[i])];
    if (n_new[i] > 0 && L % p->T != 0 && is_host(entry_c(p, reqs[i], L / p->T)))
      return ELLM_ERR_NOT_RESIDENT;
  }
  int64_t need = 0;
  for (int32_t i = 0; i < n; ++i) {
    int64_t L = p->len[size_t(reqs[i])];
    need += nchunks_of(p, L + n_new[i]) - nchunks_of(p, L);
  }
  if (need > p->n_free_kv) return ELLM_ERR_NO_CHUNKS;
  for (int32_t i = 0; i < n; ++i) {
    int32_t r = reqs[i];
    int64_t L = p->len[size_t(r)];
    for (int64_t ci = nchunks_of(p, L); ci < nchunks_of(p, L + n_new[i]); ++ci) {
      int64_t c = take_lowest_free_kv(p);
      p->chunk_req[size_t(c)] = r;
      p->chunk_idx[size_t(c)] = int32_t(ci);
      set_entry(p, r, ci, int32_t(c));
      if (p->has_dev && wait_freed(p, p->chunk_ev, c, S(stream)) != cudaSuccess) return ELLM_ERR_CUDA;
    }
    p->len[size_t(r)] = L + n_new[i];
    p->pending[size_t(r)] = n_new[i];
  }
  return flush_table(p, S(stream));
}

// a3 — O3: the KV cache grows by the generated K/V.
int ellm_kv_append(ellm_pool* p, int32_t layer, int32_t n, const int32_t* reqs,
                   const int32_t* n_new, const void* k_new, const void* v_new, void* stream) {
  if (!p || n < 0 || (n > 0 && (!reqs || !n_new))) return ELLM_ERR_INVALID_ARG;
  if (layer < 0 || layer >= p->cfg.n_layers) return ELLM_ERR_OUT_OF_RANGE;
  if (!check_reqs_range(p, n, reqs)) return ELLM_ERR_OUT_OF_RANGE;
  if (has_dup(n, reqs)) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (n_new[i] != p->pending[size_t(reqs[i])]) return ELLM_ERR_INVALID_ARG;
  int64_t rows = 0;
  for (int32_t i = 0; i < n; ++i) {
    int32_t r = reqs[i];
    int64_t L = p->len[size_t(r)];
    if (n_new[i] > 0)
      for (int64_t ci = (L - n_new[i]) / p->T; ci <= (L - 1) / p->T; ++ci)
        if (!is_dev(entry_c(p, r, ci))) return ELLM_ERR_NOT_RESIDENT;
    rows += n_new[i];
  }
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  if (rows == 0) return ELLM_OK;
  if (!k_new || !v_new) return ELLM_ERR_INVALID_ARG;
  std::vector<int32_t> d(size_t(3 * n + 1));
  int32_t cum = 0;
  for (int32_t i = 0; i < n; ++i) {
    d[size_t(i)] = reqs[i];
    d[size_t(n + i)] = int32_t(p->len[size_t(reqs[i])] - n_new[i]);
    d[size_t(2 * n + i)] = cum;
    cum += n_new[i];
  }
  d[size_t(3 * n)] = cum;
  const int32_t* dd;
  int rc = upload_ints(p, d, S(stream), &dd, nullptr);
  if (rc) return rc;
  AppendDesc ad{dd, dd + n, dd + 2 * n};
  cudaError_t e = launch_kv_append(ad, n, rows, p->d_table, p->cfg.max_chunks_per_request,
                                   static_cast<uint8_t*>(ellm_vtensor_base(p->vt)), p->chunk_bytes,
                                   p->T, layer, p->cfg.n_heads_kv, p->cfg.head_dim, k_new, v_new,
                                   p->num_sms, S(stream), p->ash.rot);
  if (e != cudaSuccess) return cuda_fail(p, e);
  ++p->launches;
  return p->ring.commit(S(stream));
}

// a4 + a5 — O4: exact softmax attention over the accumulated KV.
static int attention_impl(ellm_pool* p, int32_t layer, int32_t n, const int32_t* reqs, const void* q,
                          void* out, float scale, void* stream, const void* k_new, const void* v_new,
                          int64_t gather_off = -1);

int ellm_paged_decode_attention(ellm_pool* p, int32_t layer, int32_t n, const int32_t* reqs,
                                const void* q, void* out, float scale, void* stream) {
  if (!p || n < 0 || (n > 0 && !reqs)) return ELLM_ERR_INVALID_ARG;
  if (layer < 0 || layer >= p->cfg.n_layers) return ELLM_ERR_OUT_OF_RANGE;
  if (!check_reqs_range(p, n, reqs)) return ELLM_ERR_OUT_OF_RANGE;
  for (int32_t i = 0; i < n; ++i)
    if (p->len[size_t(reqs[i])] == 0) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (p->nonres[size_t(reqs[i])] > 0) return ELLM_ERR_NOT_RESIDENT;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  if (n == 0) return ELLM_OK;
  return attention_impl(p, layer, n, reqs, q, out, scale, stream, nullptr, nullptr);
}

// a3 + a4 + a5 fused for decode: kv_append of one token per request, then attention.
int ellm_decode_append_attention(ellm_pool* p, int32_t layer, int32_t n, const int32_t* reqs,
                                 const void* k_new, const void* v_new, const void* q, void* out,
                                 float scale, void* stream) {
  if (!p || n < 0 || (n > 0 && !reqs)) return ELLM_ERR_INVALID_ARG;
  if (layer < 0 || layer >= p->cfg.n_layers) return ELLM_ERR_OUT_OF_RANGE;
  if (!check_reqs_range(p, n, reqs)) return ELLM_ERR_OUT_OF_RANGE;
  if (has_dup(n, reqs)) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (p->pending[size_t(reqs[i])] != 1) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (p->nonres[size_t(reqs[i])] > 0) return ELLM_ERR_NOT_RESIDENT;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  if (n == 0) return ELLM_OK;
  if (!k_new || !v_new) return ELLM_ERR_INVALID_ARG;
  return attention_impl(p, layer, n, reqs, q, out, scale, stream, k_new, v_new);
}

// ---- a10: head-sharded output gather fused into the attention epilogue over peer memory ----
int ellm_gather_window_create(int32_t device, int64_t bytes, void** window_out, void* ipc_handle_out) {
  if (!window_out || bytes <= ELLM_GATHER_DATA_OFFSET || device < 0) return ELLM_ERR_INVALID_ARG;
  *window_out = nullptr;
  cudaError_t e;
  void* w = nullptr;
  if ((e = cudaSetDevice(device)) != cudaSuccess || (e = cudaMalloc(&w, size_t(bytes))) != cudaSuccess)
    return cuda_fail(nullptr, e);
  if ((e = cudaMemset(w, 0, size_t(bytes))) != cudaSuccess ||
      (ipc_handle_out && (e = cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(ipc_handle_out), w)) !=
                             cudaSuccess) ||
      (e = cudaDeviceSynchronize()) != cudaSuccess) {
    cudaFree(w);
    return cuda_fail(nullptr, e);
  }
  *window_out = w;
  return ELLM_OK;
}

int ellm_gather_window_destroy(void* window) {
  if (!window) return ELLM_ERR_INVALID_ARG;
  return cudaFree(window) == cudaSuccess ? ELLM_OK : ELLM_ERR_CUDA;
}

int ellm_ipc_open(const void* ipc_handle, void** window_out) {
  if (!ipc_handle || !window_out) return ELLM_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(window_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e == cudaSuccess) return ELLM_OK;
  cudaGetLastError();  // not sticky: clear it
  return ELLM_ERR_PEER;
}

int ellm_ipc_close(void* window) {
  if (!window) return ELLM_ERR_INVALID_ARG;
  return cudaIpcCloseMemHandle(window) == cudaSuccess ? ELLM_OK : ELLM_ERR_CUDA;
}

int ellm_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (!dst || !src || bytes < 0) return ELLM_ERR_INVALID_ARG;
  if (bytes == 0) return ELLM_OK;
  return cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDefault, S(stream)) == cudaSuccess ? ELLM_OK
                                                                                                 : ELLM_ERR_CUDA;
}

int ellm_gather_attach(ellm_pool* p, int32_t world, int32_t rank, int32_t heads_q_total,
                       void* const* windows, int64_t window_bytes) {
  if (!p || !windows) return ELLM_ERR_INVALID_ARG;
  if (world < 1 || world > ellm::kMaxPeers || rank < 0 || rank >= world) return ELLM_ERR_OUT_OF_RANGE;
  if (heads_q_total != world * p->cfg.n_heads_q || window_bytes <= ELLM_GATHER_DATA_OFFSET ||
      p->cfg.n_layers > ELLM_GATHER_DATA_OFFSET / 4)
    return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < world; ++i)
    if (!windows[i] || reinterpret_cast<uintptr_t>(windows[i]) % 256) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  // this rank's flags as they stand (zero for a fresh window): all ranks must be idle here
  std::vector<uint32_t> cur(size_t(p->cfg.n_layers));
  cudaError_t e = cudaMemcpy(cur.data(), windows[rank], cur.size() * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(p, e);
  p->g_world = world;
  p->g_rank = rank;
  p->g_hq_out = heads_q_total;
  p->g_win.assign(reinterpret_cast<uint8_t* const*>(windows), reinterpret_cast<uint8_t* const*>(windows) + world);
  p->g_win_bytes = window_bytes;
  p->g_expect = cur;
  if (const char* t = std::getenv("ELLM_GATHER_TIMEOUT_MS")) p->g_timeout_ns = uint64_t(std::atoll(t)) * 1000000ull;
  return ELLM_OK;
}

int ellm_gather_detach(ellm_pool* p) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  p->g_world = 0;
  p->g_win.clear();
  p->g_expect.clear();
  p->g_wait_flag = nullptr;
  return ELLM_OK;
}

int ellm_attention_gather(ellm_pool* p, int32_t layer, int32_t n, const int32_t* reqs, const void* k_new,
                          const void* v_new, const void* q, int64_t out_offset, float scale, void* stream) {
  if (!p || n < 0 || (n > 0 && !reqs)) return ELLM_ERR_INVALID_ARG;
  if (layer < 0 || layer >= p->cfg.n_layers) return ELLM_ERR_OUT_OF_RANGE;
  if (!check_reqs_range(p, n, reqs)) return ELLM_ERR_OUT_OF_RANGE;
  if (p->g_world == 0 || out_offset < 0 || out_offset % 16) return ELLM_ERR_INVALID_ARG;
  const int64_t rows_bytes = int64_t(n) * p->g_hq_out * p->cfg.head_dim * 2;
  if (out_offset + rows_bytes > p->g_win_bytes - ELLM_GATHER_DATA_OFFSET) return ELLM_ERR_OUT_OF_RANGE;
  if (k_new || v_new) {  // fused decode append: as ellm_decode_append_attention
    if (has_dup(n, reqs) || !k_new || !v_new) return ELLM_ERR_INVALID_ARG;
    for (int32_t i = 0; i < n; ++i)
      if (p->pending[size_t(reqs[i])] != 1) return ELLM_ERR_INVALID_ARG;
  } else {
    for (int32_t i = 0; i < n; ++i)
      if (p->len[size_t(reqs[i])] == 0) return ELLM_ERR_INVALID_ARG;
  }
  for (int32_t i = 0; i < n; ++i)
    if (p->nonres[size_t(reqs[i])] > 0) return ELLM_ERR_NOT_RESIDENT;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  if (n == 0) return ELLM_OK;
  return attention_impl(p, layer, n, reqs, q, p->g_win[size_t(p->g_rank)] + ELLM_GATHER_DATA_OFFSET + out_offset,
                        scale, stream, k_new, v_new, out_offset);
}

int ellm_gather_wait(ellm_pool* p, int32_t layer, void* stream) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  if (layer < 0 || layer >= p->cfg.n_layers) return ELLM_ERR_OUT_OF_RANGE;
  if (p->g_world == 0) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  const uint32_t* flag = reinterpret_cast<const uint32_t*>(p->g_win[size_t(p->g_rank)]) + layer;
  cudaError_t e = launch_gather_wait(flag, p->g_expect[size_t(layer)], p->g_timeout_ns, S(stream));
  if (e != cudaSuccess) return cuda_fail(p, e);
  ++p->launches;
  return ELLM_OK;
}

// a10, folded: the next attention launch of this pool waits in its producer for `layer`'s gather
// (the target the flag must reach is fixed now), so no wait kernel sits between two attention
// launches and programmatic dependent launch stays on at N > 1.
int ellm_gather_wait_next(ellm_pool* p, int32_t layer) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  if (layer < 0 || layer >= p->cfg.n_layers) return ELLM_ERR_OUT_OF_RANGE;
  if (p->g_world == 0) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  p->g_wait_flag = reinterpret_cast<const uint32_t*>(p->g_win[size_t(p->g_rank)]) + layer;
  p->g_wait_target = p->g_expect[size_t(layer)];
  return ELLM_OK;
}

}  // extern "C"

static int attention_impl(ellm_pool* p, int32_t layer, int32_t n, const int32_t* reqs, const void* q,
                          void* out, float scale, void* stream, const void* k_new, const void* v_new,
                          int64_t gather_off) {
  if (!q || !out || !std::isfinite(scale)) return ELLM_ERR_INVALID_ARG;
  if (n > p->attn_cap) {  // a list longer than max_requests (repeated ids): grow the split-K state
    const int rc = alloc_attn_state(p, std::max<int64_t>(n, 2 * p->attn_cap));
    if (rc) return rc;
  }
  const AttnShape& a = p->ash;
  const int32_t n_vr = n * a.HG;
  // descriptor cache: the same batch is attended at every layer of a decode step
  std::vector<int32_t> key(size_t(2 * n));
  for (int32_t i = 0; i < n; ++i) {
    key[size_t(i)] = reqs[i];
    key[size_t(n + i)] = int32_t(p->len[size_t(reqs[i])]);
  }
  const bool upload = key != p->cache_key || p->cache_epoch != p->table_epoch ||
                      !p->ring.still_valid(p->cache_dev, p->cache_gen);
  if (upload) {
    // layout: req[n] len[n] cum_s[n_vr+1] cum_d[n_vr+1] b_first[n_vr] b_last[n_vr]
    //         u_first[n_vr] u_last[n_vr] dyn_info[n_dyn][8] dyn_ent[n_dyn][U * npieces]
    std::vector<int32_t> d(size_t(2 * n + 6 * n_vr + 2));
    for (int32_t i = 0; i < n; ++i) {
      d[size_t(i)] = reqs[i];
      d[size_t(n + i)] = key[size_t(n + i)];
    }
    auto tiles_of = [&](int32_t vr) { return (p->len[size_t(reqs[vr / a.HG])] + a.TT - 1) / a.TT; };
    int64_t W = 0;
    for (int32_t vr = 0; vr < n_vr; ++vr) W += tiles_of(vr);
    if (W > INT32_MAX / 2) return ELLM_ERR_UNSUPPORTED;
    // Dynamic tail only when there is enough work to balance: the last tiles(vr) / dyn_div
    // tiles of every request go to the dynamic space, in units of U <= 32 tiles (one producer
    // lane per tile of a unit).
    int64_t div = (p->dyn_div > 0 && W >= 4 * int64_t(p->num_sms)) ? p->dyn_div : 0;
    if (div) {
      int64_t wd = 0;
      for (int32_t vr = 0; vr < n_vr; ++vr) wd += tiles_of(vr) / div;
      if (wd == 0 || std::max<int64_t>(p->dyn_unit, (wd + kMaxDynUnits - 1) / kMaxDynUnits) > 32) div = 0;
    }
    int32_t* cum_s = d.data() + 2 * n;
    int32_t* cum_d = cum_s + n_vr + 1;
    int64_t Ws = 0, Wd = 0;
    for (int32_t vr = 0; vr < n_vr; ++vr) {
      const int64_t tiles = tiles_of(vr);
      const int64_t dyn = div ? tiles / div : 0;  // < tiles: every request keeps >= 1 static tile
      cum_s[vr] = int32_t(Ws);
      cum_d[vr] = int32_t(Wd);
      Ws += tiles - dyn;
      Wd += dyn;
    }
    cum_s[n_vr] = int32_t(Ws);
    cum_d[n_vr] = int32_t(Wd);
    AttnPlan& pl = p->cache_plan;
    pl.W_s = Ws;
    pl.W_d = Wd;
    // G = min(#SMs, W_s): every static CTA owns >= 1 tile, so every CTA in [b_first, b_last]
    // writes a record for vr (the merge reads exactly those).
    pl.G = int32_t(std::min<int64_t>(p->num_sms, Ws));
    pl.U = Wd ? std::max<int64_t>(p->dyn_unit, (Wd + kMaxDynUnits - 1) / kMaxDynUnits) : 1;
    pl.n_dyn = Wd ? (Wd + pl.U - 1) / pl.U : 0;
    // Static CTA b owns [B[b], B[b+1]) = [floor(b W_s / G), floor((b+1) W_s / G)) of the static
    // space (equal shares; the kernel reads its range from its per-CTA record). Dynamic unit u
    // owns [u U, (u+1) U).
    const int64_t G = pl.G;
    std::vector<int64_t> B(size_t(G) + 1);
    if (int64_t(p->dbg_weights.size()) >= G) {  // measurement knob (ellm_debug_attn_weights)
      double tot = 0.0;
      for (int64_t b = 0; b < G; ++b) tot += p->dbg_weights[size_t(b)];
      double acc = 0.0;
      B[0] = 0;
      for (int64_t b = 1; b < G; ++b) {
        acc += p->dbg_weights[size_t(b - 1)];
        int64_t t = int64_t(double(Ws) * acc / tot + 0.5);
        t = std::min(std::max(t, B[size_t(b - 1)] + 1), Ws - (G - b));
        B[size_t(b)] = t;
      }
      B[size_t(G)] = Ws;
    } else {
      for (int64_t b = 0; b <= G; ++b) B[size_t(b)] = b * Ws / G;
    }
    auto cta_of = [&](int64_t t) {  // the CTA holding static tile t
      return int32_t(std::upper_bound(B.begin(), B.end(), t) - B.begin()) - 1;
    };
    int32_t* bf = cum_d + n_vr + 1;
    int32_t* bl = bf + n_vr;
    int32_t* uf = bl + n_vr;
    int32_t* ul = uf + n_vr;
    for (int32_t vr = 0; vr < n_vr; ++vr) {
      bf[vr] = cta_of(cum_s[vr]);
      bl[vr] = cta_of(int64_t(cum_s[vr + 1]) - 1);
      if (cum_d[vr + 1] > cum_d[vr]) {
        uf[vr] = int32_t(cum_d[vr] / pl.U);
        ul[vr] = int32_t((int64_t(cum_d[vr + 1]) - 1) / pl.U);
      } else {
        uf[vr] = 0;
        ul[vr] = -1;
      }
    }
    // Per dynamic unit, what the producer would otherwise look up serially: the request of its
    // first tile (+ that tile's offset in the request, the first segment's length, len, req id)
    // and the chunk ids of all its tiles, read from the host's authoritative tables.
    p->cache_info_off = (int64_t(d.size()) + 3) & ~int64_t(3);  // int4-aligned (16 B)
    const int32_t tok_box = std::min(p->T, a.TT), npieces = a.TT / tok_box;
    const int64_t U = pl.U, ulen = U * npieces;
    p->cache_ent_off = p->cache_info_off + 8 * pl.n_dyn;
    d.resize(size_t(p->cache_ent_off + pl.n_dyn * ulen), -1);
    cum_s = d.data() + 2 * n;  // (resize may have moved the buffer)
    cum_d = cum_s + n_vr + 1;
    int32_t vr = 0;
    for (int64_t u = 0; u < pl.n_dyn; ++u) {
      int32_t* info = d.data() + p->cache_info_off + 8 * u;
      int32_t* ent = d.data() + p->cache_ent_off + u * ulen;
      for (int64_t i = 0; i < U && u * U + i < Wd; ++i) {
        const int64_t t = u * U + i;
        while (cum_d[vr + 1] <= t) ++vr;
        const int32_t r = reqs[vr / a.HG];
        const int64_t len = p->len[size_t(r)];
        const int64_t tin = (cum_s[vr + 1] - cum_s[vr]) + (t - cum_d[vr]);  // tile within vr
        if (i == 0) {
          info[0] = vr;
          info[1] = int32_t(tin);
          info[2] = int32_t(cum_d[vr + 1] - t);
          info[3] = int32_t(len);
          info[4] = r;
        }
        for (int32_t k = 0; k < npieces; ++k) {
          const int64_t pos = tin * a.TT + int64_t(k) * tok_box;
          if (pos < len) ent[i * npieces + k] = entry_c(p, r, pos / p->T);
        }
      }
    }
    // Per CTA, its first static segment as the producer would look it up (a warp-wide search of
    // cum_s, then len / req / cum loads: three dependent L2 round trips before the first TMA):
    // {vr, cum_s[vr], cum_s[vr + 1], len}, {req, 0, 0, 0}.
    p->cache_cta_off = (int64_t(d.size()) + 3) & ~int64_t(3);
    d.resize(size_t(p->cache_cta_off + 8 * int64_t(pl.G)), 0);
    cum_s = d.data() + 2 * n;
    {
      int32_t v = 0;
      for (int64_t b = 0; b < pl.G; ++b) {
        const int64_t t0 = B[size_t(b)];
        while (v + 1 < n_vr && cum_s[v + 1] <= t0) ++v;
        int32_t* ci = d.data() + p->cache_cta_off + 8 * b;
        const int32_t r = reqs[v / a.HG];
        ci[0] = v;
        ci[1] = cum_s[v];
        ci[2] = cum_s[v + 1];
        ci[3] = int32_t(p->len[size_t(r)]);
        ci[4] = r;
        ci[5] = int32_t(B[size_t(b)]);      // static range [t_begin, t_end)
        ci[6] = int32_t(B[size_t(b) + 1]);
      }
    }
    const int32_t* dd;
    uint64_t gen;
    if (d.size() * 4 > p->ring.seg_bytes()) return ELLM_ERR_UNSUPPORTED;
    int rc = upload_ints(p, d, S(stream), &dd, &gen);
    if (rc) return rc;
    p->cache_key = key;
    p->cache_epoch = p->table_epoch;
    p->cache_dev = dd;
    p->cache_gen = gen;
    p->cache_n_vr = n_vr;
  } else {
    p->ring.touch(p->cache_dev);
  }
  const int32_t* dd = p->cache_dev;
  const int32_t* cs = dd + 2 * n;
  AttnDesc ad{dd, dd + n, cs, cs + n_vr + 1, cs + 2 * n_vr + 2, cs + 3 * n_vr + 2, cs + 4 * n_vr + 2,
              cs + 5 * n_vr + 2};
  AttnPlan plan = p->cache_plan;
  plan.dyn_info = dd + p->cache_info_off;
  plan.dyn_ent = dd + p->cache_ent_off;
  plan.cta_first = dd + p->cache_cta_off;
  plan.ticket = p->d_ticket;
  plan.ticket_base = p->ticket_base;
  plan.k_new = k_new;
  plan.v_new = v_new;
  plan.pool = static_cast<uint8_t*>(ellm_vtensor_base(p->vt));
  plan.chunk_bytes = p->chunk_bytes;
  if (gather_off >= 0) {  // a10: rows to every rank's window, merged counts to every rank's flag
    plan.n_peer = p->g_world;
    plan.Hq_out = p->g_hq_out;
    plan.q_off = p->g_rank * a.Hq;
    for (int32_t i = 0; i < p->g_world; ++i) {
      plan.gout[i] = p->g_win[size_t(i)] + ELLM_GATHER_DATA_OFFSET + gather_off;
      plan.gflag[i] = reinterpret_cast<uint32_t*>(p->g_win[size_t(i)]) + layer;
    }
    // the CTA that finishes last (gpu-scope count, monotone across launches) signals every rank
    plan.gdone = reinterpret_cast<uint32_t*>(p->d_ticket + 1);
    plan.gdone_target = p->gdone_base + uint32_t(plan.G);
  }
  {
    static const bool rot_ranges = [] {
      const char* v = std::getenv("ELLM_ATTN_RANGE_ROT");
      return v && std::atoi(v) != 0;
    }();
    if (rot_ranges) plan.range_shift = uint32_t((p->trace_launch * 37 + 11) % std::max<int32_t>(1, plan.G));
  }
  if (p->trace_buf) {  // ellm_set_attn_trace: this launch's [G][8] slot
    plan.trace = p->trace_buf + (p->trace_launch % p->trace_slots) * int64_t(p->num_sms) * 8;
    ++p->trace_launch;
  }
  if (p->g_wait_flag) {  // a folded gather wait (ellm_gather_wait_next) is consumed by this launch
    plan.wait_flag = p->g_wait_flag;
    plan.wait_target = p->g_wait_target;
    plan.wait_timeout_ns = p->g_timeout_ns;
    p->g_wait_flag = nullptr;
  }
  // PDL (attention.cu): only without dynamic tickets (shared counter), with a full grid (one
  // CTA per SM, so at most this launch and the previous one overlap: a third could start only
  // once all of this one's CTAs are resident, i.e. once the first has exited everywhere), and
  // when the previous launch of this pool did not append into this layer (its K/V rows may
  // still be in flight when this launch streams the layer before griddepcontrol.wait)
  // (the launch before that is also checked: under SM contention from other streams its last
  // CTA can outlive the previous launch's start-up)
  plan.pdl = p->pdl && plan.n_dyn == 0 && plan.G == p->num_sms && p->last_fused_layer != layer &&
             p->prev_fused_layer != layer;
  p->prev_fused_layer = p->last_fused_layer;
  p->last_fused_layer = k_new ? layer : -1;
  int launches = 0;
  cudaError_t e = launch_paged_attention(p->tmap, a, ad, n, n_vr, plan, p->d_table,
                                         p->cfg.max_chunks_per_request, layer, q, out, p->d_part,
                                         p->d_part_ml, p->d_arrivals, scale, S(stream), &launches);
  p->launches += launches;
  if (e != cudaSuccess) return cuda_fail(p, e);
  // tickets consumed: every unit once, plus the two outstanding tickets each CTA ends with
  if (plan.n_dyn > 0) p->ticket_base += uint64_t(plan.n_dyn) + 2 * uint64_t(plan.G);
  // every rank merges its n_vr requests once and adds them to every rank's flag word
  if (gather_off >= 0) {
    p->g_expect[size_t(layer)] += uint32_t(p->g_world) * uint32_t(n_vr);
    p->gdone_base += uint32_t(plan.G);
  }
  return upload ? p->ring.commit(S(stream)) : p->ring.commit_lazy(S(stream));
}

extern "C" {

// O8 — released slots return to the pool.
int ellm_release(ellm_pool* p, int32_t r, void* stream) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  if (r < 0 || r >= p->cfg.max_requests) return ELLM_ERR_OUT_OF_RANGE;
  int64_t nc = nchunks_of(p, p->len[size_t(r)]);
  // the request's chunks / slots are free once `stream` reaches this point
  const int32_t ev = (p->has_dev && nc > 0) ? record_free_event(p, S(stream)) : -1;
  if (p->has_dev && nc > 0 && ev < 0) return ELLM_ERR_CUDA;
  for (int64_t i = 0; i < nc; ++i) {
    int32_t e = entry_c(p, r, i);
    if (is_dev(e)) {
      if (p->off_slot[size_t(e)] >= 0) {  // an offload in progress is abandoned with the request
        free_host(p, p->off_slot[size_t(e)]);
        attach_event(p, p->slot_ev, p->off_slot[size_t(e)], ev);
        p->off_slot[size_t(e)] = -1;
      }
      free_chunk(p, e);
      attach_event(p, p->chunk_ev, e, ev);
    }
    if (is_host(e)) {
      free_host(p, host_of(e));
      attach_event(p, p->slot_ev, host_of(e), ev);
    }
    entry(p, r, i) = UNMAPPED;  // device mirror rows beyond len are never read
  }
  ++p->table_epoch;
  p->len[size_t(r)] = 0;
  p->pending[size_t(r)] = 0;
  p->nonres[size_t(r)] = 0;
  if (p->alias.count(r)) ellm_unalias_request(p, r);
  return ELLM_OK;
}

// a6 — O5: offload to CPU DRAM; deflation is the reverse of inflation.
int ellm_deflate(ellm_pool* p, int32_t n, const int32_t* ids, int32_t* slots_out, void* stream) {
  if (!p || n < 0 || (n > 0 && (!ids || !slots_out))) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= p->cfg.max_chunks) return ELLM_ERR_OUT_OF_RANGE;
  if (has_dup(n, ids)) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (p->owner[size_t(ids[i])] != KV || !p->used[size_t(ids[i])]) return ELLM_ERR_NOT_MAPPED;
  for (int32_t i = 0; i < n; ++i)
    if (p->off_slot[size_t(ids[i])] >= 0) return ELLM_ERR_IN_USE;  // layer-wise offload in progress
  if (n > p->cfg.host_slots - p->n_host_used) return ELLM_ERR_HOST_FULL;
  std::vector<int32_t> src(static_cast<size_t>(n)), dst(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    int64_t c = ids[i];
    int64_t h = take_lowest_free_host(p);
    int32_t r = p->chunk_req[size_t(c)], ci = p->chunk_idx[size_t(c)];
    p->slot_req[size_t(h)] = r;
    p->slot_idx[size_t(h)] = ci;
    set_entry(p, r, ci, enc_host(h));
    ++p->nonres[size_t(r)];
    free_chunk(p, c);
    slots_out[i] = int32_t(h);
    src[size_t(i)] = int32_t(c);
    dst[size_t(i)] = int32_t(h);
  }
  if (!p->has_dev || n == 0) return flush_table(p, S(stream));
  cudaError_t e;
  for (int32_t h : dst)  // a slot last read by an inflate on another stream
    if ((e = wait_freed(p, p->slot_ev, h, S(stream))) != cudaSuccess) return cuda_fail(p, e);
  uint8_t* pool = static_cast<uint8_t*>(ellm_vtensor_base(p->vt));
  if (p->swap_mode >= 1) {
    if ((e = ce_copy(p->host_slots, dst, pool, src, p->chunk_bytes, S(stream), p->ash.rot, p->ash.slab, 1)) !=
        cudaSuccess)
      return cuda_fail(p, e);
  } else {
    std::vector<int32_t> both(src);
    both.insert(both.end(), dst.begin(), dst.end());
    const int32_t* dd;
    both.push_back(0);  // the copy kernel's work-claim counter
  int rc = upload_ints(p, both, S(stream), &dd, nullptr);
    if (rc) return rc;
    uint8_t* hdev = nullptr;
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&hdev), p->host_slots, 0)) != cudaSuccess)
      return cuda_fail(p, e);
    if ((e = launch_chunk_copy(hdev, dd + n, pool, dd, n, p->chunk_bytes, host_copy_grid(p), work_word(dd, 2 * n), S(stream),
                               0, -1, p->ash.rot, p->ash.slab, true, false)) != cudaSuccess)
      return cuda_fail(p, e);
    ++p->launches;
  }
  {  // the source chunks are free once the copy-out on `stream` is done
    const int32_t ev = record_free_event(p, S(stream));
    if (ev < 0) return ELLM_ERR_CUDA;
    for (int32_t c : src) attach_event(p, p->chunk_ev, c, ev);
  }
  return flush_table(p, S(stream));
}

// a7 — O6: fetch when decoding is scheduled, remap onto chunks.
int ellm_inflate(ellm_pool* p, int32_t n, const int32_t* slots, int32_t* ids_out, void* stream) {
  if (!p || n < 0 || (n > 0 && (!slots || !ids_out))) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (slots[i] < 0 || slots[i] >= p->cfg.host_slots) return ELLM_ERR_OUT_OF_RANGE;
  if (has_dup(n, slots)) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (!p->hused[size_t(slots[i])]) return ELLM_ERR_NOT_MAPPED;
  if (n > p->n_free_kv) return ELLM_ERR_NO_CHUNKS;
  std::vector<int32_t> src(static_cast<size_t>(n)), dst(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    int64_t h = slots[i];
    int64_t c = take_lowest_free_kv(p);
    int32_t r = p->slot_req[size_t(h)], ci = p->slot_idx[size_t(h)];
    p->chunk_req[size_t(c)] = r;
    p->chunk_idx[size_t(c)] = ci;
    set_entry(p, r, ci, int32_t(c));
    --p->nonres[size_t(r)];
    free_host(p, h);
    ids_out[i] = int32_t(c);
    src[size_t(i)] = int32_t(h);
    dst[size_t(i)] = int32_t(c);
  }
  if (!p->has_dev || n == 0) return flush_table(p, S(stream));
  cudaError_t e;
  for (int32_t c : dst)  // a chunk freed by work on another stream
    if ((e = wait_freed(p, p->chunk_ev, c, S(stream))) != cudaSuccess) return cuda_fail(p, e);
  uint8_t* pool = static_cast<uint8_t*>(ellm_vtensor_base(p->vt));
  if (p->swap_mode == 3) {
    if ((e = side_inflate_copy(p, pool, dst, src, S(stream))) != cudaSuccess) return cuda_fail(p, e);
  } else if (p->swap_mode == 1) {
    if ((e = ce_copy(pool, dst, p->host_slots, src, p->chunk_bytes, S(stream), p->ash.rot, p->ash.slab, 2)) !=
        cudaSuccess)
      return cuda_fail(p, e);
  } else if (p->swap_mode == 2) {
    // staged: the host link writes into a device staging buffer outside the KV pool (copy
    // engines), then an SM copy moves each batch into its chunks — inbound PCIe writes into the
    // pool's VA slow a concurrent decode far more than device-side writes do (DESIGN.md §5 C3)
    const int64_t S_chunks = std::max<int64_t>(1, (int64_t(256) << 20) / p->chunk_bytes);
    if (!p->d_stage) {
      if ((e = cudaMalloc(reinterpret_cast<void**>(&p->d_stage), size_t(S_chunks * p->chunk_bytes))) != cudaSuccess)
        return cuda_fail(p, e);
      if ((e = cudaEventCreateWithFlags(&p->stage_ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(p, e);
    }
    if (p->stage_stream && p->stage_stream != S(stream) &&
        (e = cudaStreamWaitEvent(S(stream), p->stage_ev, 0)) != cudaSuccess)
      return cuda_fail(p, e);
    for (int32_t b0 = 0; b0 < n; b0 += int32_t(S_chunks)) {
      const int32_t k = int32_t(std::min<int64_t>(S_chunks, n - b0));
      std::vector<int32_t> sidx(static_cast<size_t>(k));
      std::vector<int32_t> hs(src.begin() + b0, src.begin() + b0 + k);
      for (int32_t i = 0; i < k; ++i) sidx[size_t(i)] = i;
      if ((e = ce_copy(p->d_stage, sidx, p->host_slots, hs, p->chunk_bytes, S(stream))) != cudaSuccess)
        return cuda_fail(p, e);
      std::vector<int32_t> both(sidx);
      both.insert(both.end(), dst.begin() + b0, dst.begin() + b0 + k);
      both.push_back(0);  // the copy kernel's work-claim counter
      const int32_t* dd;
      int rc = upload_ints(p, both, S(stream), &dd, nullptr);
      if (rc) return rc;
      if ((e = launch_chunk_copy(pool, dd + k, p->d_stage, dd, k, p->chunk_bytes, 2 * p->num_sms,
                                 work_word(dd, 2 * k), S(stream), 0, -1, p->ash.rot, p->ash.slab, false, true)) !=
          cudaSuccess)
        return cuda_fail(p, e);
      ++p->launches;
    }
    if ((e = cudaEventRecord(p->stage_ev, S(stream))) != cudaSuccess) return cuda_fail(p, e);
    p->stage_stream = S(stream);
  } else {
    std::vector<int32_t> both(src);
    both.insert(both.end(), dst.begin(), dst.end());
    const int32_t* dd;
    both.push_back(0);  // the copy kernel's work-claim counter
  int rc = upload_ints(p, both, S(stream), &dd, nullptr);
    if (rc) return rc;
    uint8_t* hdev = nullptr;
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&hdev), p->host_slots, 0)) != cudaSuccess)
      return cuda_fail(p, e);
    if ((e = launch_chunk_copy(pool, dd + n, hdev, dd, n, p->chunk_bytes, host_copy_grid(p), work_word(dd, 2 * n), S(stream),
                               0, -1, p->ash.rot, p->ash.slab, false, true)) != cudaSuccess)
      return cuda_fail(p, e);
    ++p->launches;
  }
  {  // the source host slots are free once the copy-in on `stream` is done
    const int32_t ev = record_free_event(p, S(stream));
    if (ev < 0) return ELLM_ERR_CUDA;
    for (int32_t h : src) attach_event(p, p->slot_ev, h, ev);
  }
  return flush_table(p, S(stream));
}

// f2 — layer-wise pipelined offload during prefill. Same end state as deflate (O5).
int ellm_offload_begin(ellm_pool* p, int32_t n, const int32_t* ids, int32_t* slots_out) {
  if (!p || n < 0 || (n > 0 && (!ids || !slots_out))) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= p->cfg.max_chunks) return ELLM_ERR_OUT_OF_RANGE;
  if (has_dup(n, ids)) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (p->owner[size_t(ids[i])] != KV || !p->used[size_t(ids[i])]) return ELLM_ERR_NOT_MAPPED;
  for (int32_t i = 0; i < n; ++i)
    if (p->off_slot[size_t(ids[i])] >= 0) return ELLM_ERR_ALREADY_MAPPED;
  if (n > p->cfg.host_slots - p->n_host_used) return ELLM_ERR_HOST_FULL;
  for (int32_t i = 0; i < n; ++i) {
    const int64_t c = ids[i], h = take_lowest_free_host(p);
    p->slot_req[size_t(h)] = p->chunk_req[size_t(c)];
    p->slot_idx[size_t(h)] = p->chunk_idx[size_t(c)];
    p->off_slot[size_t(c)] = int32_t(h);
    std::fill_n(p->off_layers.begin() + c * p->off_words, p->off_words, uint64_t(0));
    slots_out[i] = int32_t(h);
  }
  return ELLM_OK;
}

int ellm_offload_layer(ellm_pool* p, int32_t layer, int32_t n, const int32_t* ids, void* stream) {
  if (!p || n < 0 || (n > 0 && !ids)) return ELLM_ERR_INVALID_ARG;
  if (layer < 0 || layer >= p->cfg.n_layers) return ELLM_ERR_OUT_OF_RANGE;
  for (int32_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= p->cfg.max_chunks) return ELLM_ERR_OUT_OF_RANGE;
  if (has_dup(n, ids)) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (p->off_slot[size_t(ids[i])] < 0) return ELLM_ERR_NOT_MAPPED;
  std::vector<int32_t> both(size_t(2 * n));
  for (int32_t i = 0; i < n; ++i) {
    both[size_t(i)] = ids[i];
    both[size_t(n + i)] = p->off_slot[size_t(ids[i])];
  }
  // layer `layer` of each listed chunk is marked copied only once its copy is enqueued
  auto mark_copied = [&]() {
    for (int32_t i = 0; i < n; ++i)
      p->off_layers[size_t(int64_t(ids[i]) * p->off_words + layer / 64)] |= uint64_t(1) << (layer % 64);
  };
  if (!p->has_dev || n == 0) {
    mark_copied();
    return ELLM_OK;
  }
  cudaError_t e;
  for (int32_t i = 0; i < n; ++i)  // the reserved slot may have been read by an inflate elsewhere
    if ((e = wait_freed(p, p->slot_ev, both[size_t(n + i)], S(stream))) != cudaSuccess) return cuda_fail(p, e);
  // layer l's K and V slabs of all local heads: [2][Hkv][T][d] bf16, contiguous in the chunk
  const int64_t seg = int64_t(4) * p->cfg.n_heads_kv * p->T * p->cfg.head_dim;
  uint8_t* pool = static_cast<uint8_t*>(ellm_vtensor_base(p->vt));
  if (p->swap_mode >= 1) {  // copy engines (no SMs taken from the prefill compute)
    std::vector<CopyPiece> pc(static_cast<size_t>(n));
    for (int32_t i = 0; i < n; ++i) {
      const int64_t c = ids[i], h = both[size_t(n + i)];
      pc[size_t(i)] = {p->host_slots + h * p->chunk_bytes + int64_t(layer) * seg,
                       pool + c * p->chunk_bytes + int64_t(slab_slot(c, layer, p->ash.rot)) * seg, seg};
    }
    if ((e = issue_copies(pc, S(stream))) != cudaSuccess) return cuda_fail(p, e);
    mark_copied();
    return ELLM_OK;
  }
  const int32_t* dd;
  both.push_back(0);  // the copy kernel's work-claim counter
  int rc = upload_ints(p, both, S(stream), &dd, nullptr);
  if (rc) return rc;
  uint8_t* hdev = nullptr;
  if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&hdev), p->host_slots, 0)) != cudaSuccess)
    return cuda_fail(p, e);
  if ((e = launch_chunk_copy(hdev, dd + n, pool, dd, n, p->chunk_bytes,
                             host_copy_grid(p), work_word(dd, 2 * n), S(stream), int64_t(layer) * seg, seg,
                             p->ash.rot, p->ash.slab, true, false)) != cudaSuccess)
    return cuda_fail(p, e);
  ++p->launches;
  mark_copied();
  return p->ring.commit(S(stream));
}

int ellm_offload_commit(ellm_pool* p, int32_t n, const int32_t* ids, void* stream) {
  if (!p || n < 0 || (n > 0 && !ids)) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= p->cfg.max_chunks) return ELLM_ERR_OUT_OF_RANGE;
  if (has_dup(n, ids)) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (p->off_slot[size_t(ids[i])] < 0) return ELLM_ERR_NOT_MAPPED;
  for (int32_t i = 0; i < n; ++i)
    for (int32_t l = 0; l < p->cfg.n_layers; ++l)
      if (!((p->off_layers[size_t(int64_t(ids[i]) * p->off_words + l / 64)] >> (l % 64)) & 1))
        return ELLM_ERR_INVALID_ARG;  // a layer of this chunk was never copied
  const int32_t ev = p->has_dev && n > 0 ? record_free_event(p, S(stream)) : -1;
  if (p->has_dev && n > 0 && ev < 0) return ELLM_ERR_CUDA;
  for (int32_t i = 0; i < n; ++i) {
    const int64_t c = ids[i], h = p->off_slot[size_t(c)];
    const int32_t r = p->chunk_req[size_t(c)], ci = p->chunk_idx[size_t(c)];
    set_entry(p, r, ci, enc_host(h));
    ++p->nonres[size_t(r)];
    p->off_slot[size_t(c)] = -1;
    free_chunk(p, c);
    attach_event(p, p->chunk_ev, c, ev);  // free once the copies on `stream` are done
  }
  return flush_table(p, S(stream));
}

// a8 — O7: D2D migration (BJ north_star; the paper's own migration is ownership-only).
int ellm_migrate(ellm_pool* p, int32_t n, const int32_t* src, const int32_t* dst, void* stream) {
  if (!p || n < 0 || (n > 0 && (!src || !dst))) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (src[i] < 0 || src[i] >= p->cfg.max_chunks) return ELLM_ERR_OUT_OF_RANGE;
  for (int32_t i = 0; i < n; ++i)
    if (dst[i] < 0 || dst[i] >= p->cfg.max_chunks) return ELLM_ERR_OUT_OF_RANGE;
  std::vector<int32_t> all(src, src + n);
  all.insert(all.end(), dst, dst + n);
  if (has_dup(int32_t(all.size()), all.data())) return ELLM_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (p->owner[size_t(src[i])] != KV || !p->used[size_t(src[i])]) return ELLM_ERR_NOT_MAPPED;
  for (int32_t i = 0; i < n; ++i)
    if (p->off_slot[size_t(src[i])] >= 0) return ELLM_ERR_IN_USE;  // layer-wise offload in progress
  for (int32_t i = 0; i < n; ++i) {
    if (p->owner[size_t(dst[i])] != KV) return ELLM_ERR_NOT_MAPPED;
    if (p->used[size_t(dst[i])]) return ELLM_ERR_ALREADY_MAPPED;
  }
  for (int32_t i = 0; i < n; ++i) {
    int64_t s = src[i], d = dst[i];
    int32_t r = p->chunk_req[size_t(s)], ci = p->chunk_idx[size_t(s)];
    p->used[size_t(d)] = 1;
    --p->n_free_kv;
    ++p->n_used_kv;
    p->chunk_req[size_t(d)] = r;
    p->chunk_idx[size_t(d)] = ci;
    set_entry(p, r, ci, int32_t(d));
    free_chunk(p, s);
  }
  if (!p->has_dev || n == 0) return flush_table(p, S(stream));
  cudaError_t e;
  for (int32_t i = 0; i < n; ++i)  // destinations freed by work on another stream
    if ((e = wait_freed(p, p->chunk_ev, dst[i], S(stream))) != cudaSuccess) return cuda_fail(p, e);
  const int32_t* dd;
  all.push_back(0);  // the copy kernel's work-claim counter
  int rc = upload_ints(p, all, S(stream), &dd, nullptr);
  if (rc) return rc;
  uint8_t* pool = static_cast<uint8_t*>(ellm_vtensor_base(p->vt));
  e = launch_chunk_copy(pool, dd + n, pool, dd, n, p->chunk_bytes, 2 * p->num_sms, work_word(dd, 2 * n), S(stream), 0,
                        -1, p->ash.rot, p->ash.slab, true, true);
  if (e != cudaSuccess) return cuda_fail(p, e);
  ++p->launches;
  {  // the source chunks are free once the copy on `stream` is done
    const int32_t ev = record_free_event(p, S(stream));
    if (ev < 0) return ELLM_ERR_CUDA;
    for (int32_t i = 0; i < n; ++i) attach_event(p, p->chunk_ev, src[i], ev);
  }
  return flush_table(p, S(stream));
}

// a9 — inflation (3)-(4): ACT -> KV ownership transfer + on-demand remap. Chunks
// inside live activation slots are not reclaimable (only inactive eTensor memory).
// Units activations used are still mapped (f3), and with f1 the next units are pre-mapped, so
// the usual grow makes no driver call; otherwise units are mapped here (map_units_now).
int ellm_pool_grow(ellm_pool* p, int64_t n) {
  if (!p || n < 0) return ELLM_ERR_INVALID_ARG;
  if (n > p->n_act - p->n_act_used) return ELLM_ERR_NO_CHUNKS;
  std::vector<int64_t> ids;
  for (int64_t c = 0; c < p->cfg.max_chunks && int64_t(ids.size()) < n; ++c)
    if (p->owner[size_t(c)] == ACT && !p->in_act[size_t(c)]) ids.push_back(c);
  std::unique_lock<std::mutex> lk(p->vmm_mu, std::defer_lock);
  if (p->has_dev) {  // map first so a driver failure leaves ownership unchanged
    lk.lock();
    const int64_t t0 = now_ns();
    std::set<int64_t> units;
    for (int64_t c : ids) units.insert(c / p->chunks_per_unit);
    for (int64_t u : units)
      if (p->vt->mapped[size_t(u)] && !p->doomed[size_t(u)] && p->unit_kv[size_t(u)] == 0) ++p->premap_hits;
    int rc = map_units_now(p, units, units);
    p->crit_vmm_ns += now_ns() - t0;
    if (rc) return rc;
  }
  for (int64_t c : ids) {
    p->owner[size_t(c)] = KV;
    p->used[size_t(c)] = 0;
    if (p->has_dev) {
      const size_t u = size_t(c / p->chunks_per_unit);
      if (!unit_live(p, u)) ++p->unit_gen[u];
      ++p->unit_kv[u];
      p->act_cached[u] = 0;  // the memory now belongs to the KV pool
    }
    ++p->n_free_kv;
    --p->n_act;
    p->free_hint = std::min(p->free_hint, c);
  }
  if (p->has_dev) vmm_kick(p);  // refill the premap window
  return ELLM_OK;
}

// a9 — deflation, "the reverse process": highest-id FREE KV chunks -> ACT, and
// physical memory whose chunks are all ACT is unmapped — here, device-synchronising,
// unless f1's asynchronous unmapping hands it to the worker; units inside the premap window
// stay mapped either way.
int ellm_pool_shrink(ellm_pool* p, int64_t n) {
  if (!p || n < 0) return ELLM_ERR_INVALID_ARG;
  if (n > p->n_free_kv) return ELLM_ERR_IN_USE;
  std::unique_lock<std::mutex> lk(p->vmm_mu, std::defer_lock);
  if (p->has_dev) lk.lock();
  std::vector<int64_t> units;
  for (int64_t c = p->cfg.max_chunks - 1; c >= 0 && n > 0; --c)
    if (p->owner[size_t(c)] == KV && !p->used[size_t(c)]) {
      p->owner[size_t(c)] = ACT;
      --p->n_free_kv;
      ++p->n_act;
      --n;
      int64_t u = c / p->chunks_per_unit;
      if (p->has_dev && --p->unit_kv[size_t(u)] == 0 && !unit_live(p, size_t(u))) units.push_back(u);
    }
  if (!p->has_dev) return ELLM_OK;
  if (!p->async_unmap && !units.empty()) {
    const int64_t t0 = now_ns();
    int rc = unmap_units_now(p, units);
    p->crit_vmm_ns += now_ns() - t0;
    if (rc) return rc;
  }
  vmm_kick(p);
  return ELLM_OK;
}

// ---- f3: activation eTensors in the unified pool ------------------------------
// O10: a slot of ceil(bytes / chunk_bytes) consecutive idle ACT chunks, the run with the highest
// last id (activations fill the pool from the top; KV inflation takes the lowest ids).
int ellm_act_alloc(ellm_pool* p, int64_t bytes, void* stream, int64_t* first_out, void** ptr_out) {
  if (!p || bytes <= 0 || !first_out) return ELLM_ERR_INVALID_ARG;
  const int64_t n = (bytes + p->chunk_bytes - 1) / p->chunk_bytes;
  int64_t first = -1, run = 0;
  for (int64_t c = p->cfg.max_chunks - 1; c >= 0; --c) {
    run = (p->owner[size_t(c)] == ACT && !p->in_act[size_t(c)]) ? run + 1 : 0;
    if (run == n) {
      first = c;
      break;
    }
  }
  if (first < 0) return ELLM_ERR_NO_CHUNKS;
  if (p->has_dev) {
    std::lock_guard<std::mutex> g(p->vmm_mu);
    const int64_t t0 = now_ns();
    std::set<int64_t> units;
    for (int64_t c = first; c < first + n; ++c) units.insert(c / p->chunks_per_unit);
    int rc = map_units_now(p, units, units);
    p->crit_vmm_ns += now_ns() - t0;
    if (rc) return rc;
    for (int64_t c = first; c < first + n; ++c) {
      const size_t u = size_t(c / p->chunks_per_unit);
      if (!unit_live(p, u)) ++p->unit_gen[u];
      ++p->unit_act[u];
      p->act_cached[u] = 1;
      cudaError_t e = wait_freed(p, p->chunk_ev, c, S(stream));  // memory freed on another stream
      if (e != cudaSuccess) return cuda_fail(p, e);
    }
    vmm_kick(p);
  }
  for (int64_t c = first; c < first + n; ++c) p->in_act[size_t(c)] = 1;
  p->act_len[size_t(first)] = n;
  p->n_act_used += n;
  *first_out = first;
  if (ptr_out) *ptr_out = p->has_dev ? static_cast<uint8_t*>(ellm_vtensor_base(p->vt)) + first * p->chunk_bytes : nullptr;
  return ELLM_OK;
}

// O11: the slot starting at `first` ends; its chunks stay ACT and mapped (reclaimable by grow).
// Work on `stream` so far is the slot's last use (stream-ordered reuse, as for KV chunks).
int ellm_act_free(ellm_pool* p, int64_t first, void* stream) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  if (first < 0 || first >= p->cfg.max_chunks) return ELLM_ERR_OUT_OF_RANGE;
  const int64_t n = p->act_len[size_t(first)];
  if (n == 0) return ELLM_ERR_NOT_MAPPED;
  if (p->has_dev) {
    std::lock_guard<std::mutex> g(p->vmm_mu);
    const int32_t ev = record_free_event(p, S(stream));
    if (ev < 0) return cuda_fail(p, cudaGetLastError());
    for (int64_t c = first; c < first + n; ++c) {
      attach_event(p, p->chunk_ev, c, ev);
      --p->unit_act[size_t(c / p->chunks_per_unit)];
    }
    if (p->free_events[size_t(ev)].refs == 0) p->free_event_pool.push_back(ev);
  }
  for (int64_t c = first; c < first + n; ++c) p->in_act[size_t(c)] = 0;
  p->act_len[size_t(first)] = 0;
  p->n_act_used -= n;
  return ELLM_OK;
}

// Release the activation cache: units kept mapped only because activations used them.
int ellm_act_trim(ellm_pool* p) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev) return ELLM_OK;
  std::lock_guard<std::mutex> g(p->vmm_mu);
  std::vector<int64_t> units;
  for (size_t u = 0; u < p->act_cached.size(); ++u)
    if (p->act_cached[u] && p->unit_act[u] == 0) {
      p->act_cached[u] = 0;
      if (p->unit_kv[u] == 0) units.push_back(int64_t(u));
    }
  if (!p->async_unmap && !units.empty()) {
    const int64_t t0 = now_ns();
    int rc = unmap_units_now(p, units);
    p->crit_vmm_ns += now_ns() - t0;
    if (rc) return rc;
  }
  vmm_kick(p);
  return ELLM_OK;
}

// torch.cuda.memory.CUDAPluggableAllocator entry points (the framework's caching
// allocator keeps its BFC strategy on top; its segments come from activation slots).
static ellm_pool* g_torch_pool = nullptr;
int ellm_torch_set_pool(ellm_pool* p) {
  g_torch_pool = p;
  return ELLM_OK;
}
void* ellm_torch_alloc(size_t size, int device, void* stream) {
  ellm_pool* p = g_torch_pool;
  if (!p || !p->has_dev || device != p->cfg.device || size == 0) return nullptr;
  int64_t first = -1;
  void* ptr = nullptr;
  return ellm_act_alloc(p, int64_t(size), stream, &first, &ptr) == ELLM_OK ? ptr : nullptr;
}
void ellm_torch_free(void* ptr, size_t size, int device, void* stream) {
  (void)size;
  (void)device;
  ellm_pool* p = g_torch_pool;
  if (!p || !p->has_dev || !ptr) return;
  const int64_t off = static_cast<uint8_t*>(ptr) - static_cast<uint8_t*>(ellm_vtensor_base(p->vt));
  if (off >= 0 && off % p->chunk_bytes == 0) ellm_act_free(p, off / p->chunk_bytes, stream);
}

// ---- f4: chunked-prefill attention (prefill.cu) ------------------------------------
// Work items: (request, kv-head, block of 128/group query positions), longest first.
int ellm_prefill_attention(ellm_pool* p, int32_t layer, int32_t n, const int32_t* reqs, const int32_t* n_q,
                           const void* q, void* out, float scale, void* stream) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  if (layer < 0 || layer >= p->cfg.n_layers) return ELLM_ERR_OUT_OF_RANGE;
  if (n < 0 || (n > 0 && (!reqs || !n_q || !q || !out))) return ELLM_ERR_INVALID_ARG;
  if (!check_reqs_range(p, n, reqs)) return ELLM_ERR_OUT_OF_RANGE;
  if (128 % p->group != 0) return ELLM_ERR_UNSUPPORTED;
  int64_t rows = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int64_t len = p->len[size_t(reqs[i])];
    if (len == 0 || n_q[i] < 1 || n_q[i] > len) return ELLM_ERR_INVALID_ARG;
    rows += n_q[i];
  }
  for (int32_t i = 0; i < n; ++i)
    if (p->nonres[size_t(reqs[i])] > 0) return ELLM_ERR_NOT_RESIDENT;
  if (n == 0) return ELLM_OK;
  cudaStream_t st = S(stream);
  if (int rc = flush_table(p, st)) return rc;
  const int bp = 256 / p->group;  // query positions per work item: two Q tiles of 128 rows (prefill.cu)
  struct Item { int32_t v[8]; };
  std::vector<Item> items;
  int64_t row0 = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t r = reqs[i];
    const int64_t len = p->len[size_t(r)];
    for (int64_t b = 0; b < n_q[i]; b += bp) {
      const int64_t pos0 = len - n_q[i] + b;
      const int64_t nv = std::min<int64_t>(bp, n_q[i] - b);
      const int64_t tiles = (pos0 + nv + 127) / 128;  // 128-key tiles (prefill.cu kN) over keys 0 .. pos0 + nv - 1
      for (int32_t h = 0; h < p->cfg.n_heads_kv; ++h)
        items.push_back({{r, int32_t(len), int32_t(row0 + b), int32_t(pos0), int32_t(nv), h, int32_t(tiles), 0}});
    }
    row0 += n_q[i];
  }
  std::stable_sort(items.begin(), items.end(), [](const Item& a, const Item& b) { return a.v[6] > b.v[6]; });
  std::vector<int32_t> flat(items.size() * 8);
  for (size_t i = 0; i < items.size(); ++i) std::memcpy(&flat[i * 8], items[i].v, 32);
  const int32_t* d_work = nullptr;
  if (flat.size() * 4 > p->ring.seg_bytes()) return ELLM_ERR_UNSUPPORTED;  // > 32K work items
  if (int rc = upload_ints(p, flat, st, &d_work, nullptr)) return rc;
  cudaError_t e;
  if (!p->pf_ready) {
    if ((e = encode_prefill_kv_maps(&p->pf_maps, ellm_vtensor_base(p->vt), p->cfg.max_chunks, p->ash,
                                    p->chunk_bytes)) != cudaSuccess)
      return cuda_fail(p, e);
    p->pf_ready = true;
  }
  if ((e = encode_prefill_q_map(&p->pf_maps, p->ash, q, rows)) != cudaSuccess) return cuda_fail(p, e);
  e = launch_prefill_attention(p->pf_maps, p->ash, d_work, int32_t(items.size()), p->d_table,
                               p->cfg.max_chunks_per_request, layer, out, scale, st, p->trace_buf);
  if (e != cudaSuccess) return cuda_fail(p, e);
  ++p->launches;
  return p->ring.commit(st);
}

int ellm_set_launch_overlap(ellm_pool* p, int32_t enable) {
  if (!p || (enable != 0 && enable != 1)) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  if (!p->pdl_env) p->pdl = enable != 0;
  return ELLM_OK;
}

int ellm_set_vmm_overlap(ellm_pool* p, int64_t premap_bytes, int32_t async_unmap) {
  if (!p || premap_bytes < 0 || (async_unmap != 0 && async_unmap != 1)) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  {
    std::lock_guard<std::mutex> g(p->vmm_mu);
    p->premap_units = (premap_bytes + p->unit_bytes - 1) / p->unit_bytes;
    p->async_unmap = async_unmap != 0;
    if (!p->vmm_started) {
      p->vmm_thread = std::thread(vmm_worker, p);
      p->vmm_started = true;
    }
    vmm_kick(p);
  }
  return ELLM_OK;
}

int ellm_vmm_sync(ellm_pool* p) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  if (!p->has_dev || !p->vmm_started) return ELLM_OK;
  std::unique_lock<std::mutex> lk(p->vmm_mu);
  p->vmm_cv.wait(lk, [&] { return !p->vmm_dirty && !p->vmm_busy; });
  return p->vmm_error;
}

int ellm_get_table(const ellm_pool* p, int32_t r, int32_t* entries, int32_t cap, int32_t* n_out,
                   int32_t* len_out) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  if (r < 0 || r >= p->cfg.max_requests) return ELLM_ERR_OUT_OF_RANGE;
  int64_t nc = nchunks_of(p, p->len[size_t(r)]);
  if (n_out) *n_out = int32_t(nc);
  if (len_out) *len_out = int32_t(p->len[size_t(r)]);
  for (int64_t i = 0; i < nc && i < cap; ++i) entries[i] = entry_c(p, r, i);
  return ELLM_OK;
}

int ellm_chunk_states(const ellm_pool* p, int64_t first, int64_t n, uint8_t* out) {
  if (!p || n < 0 || (n > 0 && !out)) return ELLM_ERR_INVALID_ARG;
  if (first < 0 || first + n > p->cfg.max_chunks) return ELLM_ERR_OUT_OF_RANGE;
  for (int64_t i = 0; i < n; ++i) {
    const size_t c = size_t(first + i);
    out[i] = p->owner[c] == ACT ? (p->in_act[c] ? ELLM_CHUNK_ACT_SLOT : ELLM_CHUNK_ACT)
                                : p->used[c] ? ELLM_CHUNK_USED : ELLM_CHUNK_FREE;
  }
  return ELLM_OK;
}

int ellm_read_chunk(ellm_pool* p, int64_t c, void* host_dst, void* stream) {
  if (!p || !host_dst) return ELLM_ERR_INVALID_ARG;
  if (c < 0 || c >= p->cfg.max_chunks) return ELLM_ERR_OUT_OF_RANGE;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  if (p->owner[size_t(c)] != KV) return ELLM_ERR_NOT_MAPPED;
  cudaError_t e;
  const uint8_t* src = static_cast<const uint8_t*>(ellm_vtensor_base(p->vt)) + c * p->chunk_bytes;
  // the canonical [L][2][Hkv][T][d] image: layer l from slab slot slab_slot(c, l)
  const int64_t r = slab_shift(c, p->ash.rot), sl = p->ash.slab;
  uint8_t* dst = static_cast<uint8_t*>(host_dst);
  if ((e = cudaMemcpyAsync(dst, src + r * sl, size_t(p->chunk_bytes - r * sl), cudaMemcpyDeviceToHost,
                           S(stream))) != cudaSuccess ||
      (r > 0 && (e = cudaMemcpyAsync(dst + (p->chunk_bytes - r * sl), src, size_t(r * sl), cudaMemcpyDeviceToHost,
                                     S(stream))) != cudaSuccess) ||
      (e = cudaStreamSynchronize(S(stream))) != cudaSuccess)
    return cuda_fail(p, e);
  return ELLM_OK;
}

int ellm_read_host_slot(ellm_pool* p, int64_t h, void* host_dst) {
  if (!p || !host_dst) return ELLM_ERR_INVALID_ARG;
  if (h < 0 || h >= p->cfg.host_slots) return ELLM_ERR_OUT_OF_RANGE;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(p, e);
  std::memcpy(host_dst, p->host_slots + h * p->chunk_bytes, size_t(p->chunk_bytes));
  return ELLM_OK;
}

// The paper's literal KV eTensor: the request's physical chunks mapped, in logical order,
// into one contiguous VA span, using multi-mapping of a handle.
int ellm_alias_request(ellm_pool* p, int32_t r, void** out) {
  if (!p || !out) return ELLM_ERR_INVALID_ARG;
  if (r < 0 || r >= p->cfg.max_requests) return ELLM_ERR_OUT_OF_RANGE;
  if (!p->has_dev) return ELLM_ERR_NO_DEVICE;
  if (p->chunks_per_unit != 1) return ELLM_ERR_UNSUPPORTED;
  if (p->alias.count(r)) return ELLM_ERR_ALREADY_MAPPED;
  int64_t nc = nchunks_of(p, p->len[size_t(r)]);
  if (nc == 0) return ELLM_ERR_INVALID_ARG;
  if (p->nonres[size_t(r)] > 0) return ELLM_ERR_NOT_RESIDENT;
  const Driver& d = driver();
  size_t bytes = size_t(nc) * size_t(p->chunk_bytes);
  CUdeviceptr va = 0;
  if (d.memAddressReserve(&va, bytes, size_t(p->unit_bytes), 0, 0) != CUDA_SUCCESS) return ELLM_ERR_CUDA;
  for (int64_t i = 0; i < nc; ++i) {
    int32_t c = entry_c(p, r, i);
    if (d.memMap(va + CUdeviceptr(i) * p->chunk_bytes, size_t(p->chunk_bytes), 0,
                 p->vt->handles[size_t(c)], 0) != CUDA_SUCCESS) {
      for (int64_t j = 0; j < i; ++j) d.memUnmap(va + CUdeviceptr(j) * p->chunk_bytes, size_t(p->chunk_bytes));
      d.memAddressFree(va, bytes);
      return ELLM_ERR_CUDA;
    }
  }
  CUmemAccessDesc acc;
  std::memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = p->cfg.device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (d.memSetAccess(va, bytes, &acc, 1) != CUDA_SUCCESS) return ELLM_ERR_CUDA;
  p->alias[r] = {va, bytes};
  *out = reinterpret_cast<void*>(va);
  return ELLM_OK;
}

int ellm_unalias_request(ellm_pool* p, int32_t r) {
  if (!p) return ELLM_ERR_INVALID_ARG;
  auto it = p->alias.find(r);
  if (it == p->alias.end()) return ELLM_ERR_NOT_MAPPED;
  cudaDeviceSynchronize();
  const Driver& d = driver();
  const size_t cb = size_t(p->chunk_bytes);
  for (size_t off = 0; off < it->second.second; off += cb) d.memUnmap(it->second.first + off, cb);
  d.memAddressFree(it->second.first, it->second.second);
  p->alias.erase(it);
  return ELLM_OK;
}

}  // extern "C"

// vmm.cpp — driver VMM entry points, the vtensor (the paper's eTensor) and the
// staging ring used to snapshot host metadata into stream-ordered device uploads.
#include <dlfcn.h>
#include <time.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"

namespace ellm {

int64_t now_ns() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return int64_t(t.tv_sec) * 1000000000LL + t.tv_nsec;
}

template <typename F>
static bool load_sym(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p) {
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    bool ok = true;
    ok &= load_sym("cuMemAddressReserve", d.memAddressReserve);
    ok &= load_sym("cuMemAddressFree", d.memAddressFree);
    ok &= load_sym("cuMemCreate", d.memCreate);
    ok &= load_sym("cuMemRelease", d.memRelease);
    ok &= load_sym("cuMemMap", d.memMap);
    ok &= load_sym("cuMemUnmap", d.memUnmap);
    ok &= load_sym("cuMemSetAccess", d.memSetAccess);
    ok &= load_sym("cuMemGetAllocationGranularity", d.memGetAllocationGranularity);
    ok &= load_sym("cuTensorMapEncodeTiled", d.tensorMapEncodeTiled);
    d.ok = ok;
  });
  return d;
}

// The context calls by their explicit ABI names from the driver library itself (the unversioned
// entry-point query can resolve "cuCtxCreate" to a later ABI with a different signature).
template <typename F>
static bool load_drv(void* lib, const char* name, F& fn) {
  void* p = lib ? dlsym(lib, name) : nullptr;
  fn = reinterpret_cast<F>(p);
  return p != nullptr;
}

const CtxDriver& ctx_driver() {
  static CtxDriver d;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    bool ok = lib != nullptr;
    ok &= load_drv(lib, "cuDeviceGet", d.deviceGet);
    ok &= load_drv(lib, "cuCtxCreate_v2", d.ctxCreate);
    ok &= load_drv(lib, "cuCtxDestroy_v2", d.ctxDestroy);
    ok &= load_drv(lib, "cuCtxPushCurrent_v2", d.ctxPushCurrent);
    ok &= load_drv(lib, "cuCtxPopCurrent_v2", d.ctxPopCurrent);
    d.ok = ok;
  });
  return d;
}

static CUmemAllocationProp device_prop(int device) {
  CUmemAllocationProp p;
  std::memset(&p, 0, sizeof(p));
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  return p;
}

// ---- staging ring ---------------------------------------------------------------------
int StagingRing::init(size_t seg_bytes, int n_segs) {
  seg_bytes_ = seg_bytes;
  n_segs_ = n_segs;
  if (cudaHostAlloc(reinterpret_cast<void**>(&h_), seg_bytes * n_segs, cudaHostAllocDefault) !=
      cudaSuccess)
    return ELLM_ERR_CUDA;
  if (cudaMalloc(reinterpret_cast<void**>(&d_), seg_bytes * n_segs) != cudaSuccess)
    return ELLM_ERR_CUDA;
  segs_.assign(size_t(n_segs), Seg());
  for (int i = 0; i < n_segs; ++i) segs_[size_t(i)].generation = uint64_t(i) + 1;
  cur_ = 0;
  off_ = 0;
  return ELLM_OK;
}

void StagingRing::destroy() {
  for (auto& s : segs_)
    for (auto e : s.events) cudaEventDestroy(e);
  for (auto e : free_events_) cudaEventDestroy(e);
  segs_.clear();
  free_events_.clear();
  if (h_) cudaFreeHost(h_);
  if (d_) cudaFree(d_);
  h_ = d_ = nullptr;
}

int StagingRing::retire_and_advance() {
  cur_ = (cur_ + 1) % n_segs_;
  off_ = 0;
  if (int rc = flush_pending(cur_)) return rc;
  Seg& s = segs_[size_t(cur_)];
  for (auto e : s.events) {  // the segment's previous consumers must be done
    static const bool dbg = std::getenv("ELLM_DEBUG_WAITS") != nullptr;  // measurement aid
    if (dbg && cudaEventQuery(e) == cudaErrorNotReady)
      std::fprintf(stderr, "[ellm] staging ring: host waits for segment %d's consumers\n", cur_);
    if (cudaEventSynchronize(e) != cudaSuccess) return ELLM_ERR_CUDA;
    free_events_.push_back(e);
  }
  s.events.clear();
  s.streams.clear();
  s.generation += uint64_t(n_segs_);
  return ELLM_OK;
}

int StagingRing::alloc(size_t bytes, void** host, void** dev, uint64_t* generation) {
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes > seg_bytes_) return ELLM_ERR_INVALID_ARG;
  if (off_ + bytes > seg_bytes_) {
    int rc = retire_and_advance();
    if (rc) return rc;
  }
  size_t o = size_t(cur_) * seg_bytes_ + off_;
  *host = h_ + o;
  *dev = d_ + o;
  if (generation) *generation = segs_[size_t(cur_)].generation;
  off_ += bytes;
  touch(*dev);
  return ELLM_OK;
}

void StagingRing::touch(const void* dev) {
  int seg = int(size_t(static_cast<const uint8_t*>(dev) - d_) / seg_bytes_);
  if (std::find(touched_.begin(), touched_.end(), seg) == touched_.end()) touched_.push_back(seg);
}

int StagingRing::upload(void* dev, size_t bytes, cudaStream_t stream) {
  size_t o = size_t(static_cast<uint8_t*>(dev) - d_);
  if (cudaMemcpyAsync(dev, h_ + o, bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return ELLM_ERR_CUDA;
  return ELLM_OK;
}

int StagingRing::commit(cudaStream_t stream) {
  if (int rc = flush_pending(-1)) return rc;
  for (int seg : touched_) {
    int rc = commit_seg(seg, stream);
    if (rc) return rc;
  }
  touched_.clear();
  return ELLM_OK;
}

// Work that only re-reads an uploaded segment (an attention launch whose descriptors are
// cached) records no event now — an event between two attention launches would stop the
// second from overlapping the first (PDL). The event is recorded on the same stream later:
// at the next eager commit, or before the segment is reused; it then also covers this work.
int StagingRing::commit_lazy(cudaStream_t stream) {
  for (int seg : touched_) {
    bool have = false;
    for (auto& ps : pending_) have |= (ps.first == seg && ps.second == stream);
    if (!have) pending_.emplace_back(seg, stream);
  }
  touched_.clear();
  return ELLM_OK;
}

int StagingRing::flush_pending(int only_seg) {
  for (size_t i = 0; i < pending_.size();) {
    if (only_seg >= 0 && pending_[i].first != only_seg) {
      ++i;
      continue;
    }
    if (int rc = commit_seg(pending_[i].first, pending_[i].second)) return rc;
    pending_.erase(pending_.begin() + long(i));
  }
  return ELLM_OK;
}

int StagingRing::commit_seg(int seg, cudaStream_t stream) {
  Seg& s = segs_[size_t(seg)];
  cudaEvent_t e = nullptr;
  // one event per distinct stream; re-recording captures the latest work on that stream
  for (size_t i = 0; i < s.streams.size(); ++i)
    if (s.streams[i] == stream) e = s.events[i];
  if (!e) {
    if (!free_events_.empty()) {
      e = free_events_.back();
      free_events_.pop_back();
    } else if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      return ELLM_ERR_CUDA;
    }
    s.events.push_back(e);
    s.streams.push_back(stream);
  }
  return cudaEventRecord(e, stream) == cudaSuccess ? ELLM_OK : ELLM_ERR_CUDA;
}

bool StagingRing::still_valid(const void* dev, uint64_t generation) const {
  if (!dev) return false;
  size_t o = size_t(static_cast<const uint8_t*>(dev) - d_);
  size_t seg = o / seg_bytes_;
  return seg < segs_.size() && segs_[seg].generation == generation;
}

}  // namespace ellm

using namespace ellm;

extern "C" {

int ellm_vmm_granularity(int32_t device, size_t* out) {
  if (!out || device < 0) return ELLM_ERR_INVALID_ARG;
  const Driver& d = driver();
  if (!d.ok) return ELLM_ERR_CUDA;
  CUmemAllocationProp p = device_prop(device);
  if (d.memGetAllocationGranularity(out, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS)
    return ELLM_ERR_CUDA;
  return ELLM_OK;
}

int ellm_vtensor_create(int32_t device, size_t slot_bytes, int64_t n_slots, ellm_vtensor** out) {
  if (!out || device < 0 || slot_bytes == 0 || n_slots <= 0) return ELLM_ERR_INVALID_ARG;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess)
    return ELLM_ERR_CUDA;
  size_t gran = 0;
  int rc = ellm_vmm_granularity(device, &gran);
  if (rc) return rc;
  if (slot_bytes % gran != 0) return ELLM_ERR_INVALID_ARG;
  const Driver& d = driver();
  ellm_vtensor* vt = new ellm_vtensor();
  vt->device = device;
  vt->slot_bytes = slot_bytes;
  vt->n_slots = n_slots;
  // VA aligned to the largest power of two dividing the slot (<= 1 GiB), so the driver may back
  // large slots with its large page sizes (fewer TLB entries for the attention's scattered reads)
  size_t align = gran;
  while (align < (size_t(1) << 30) && slot_bytes % (align * 2) == 0) align *= 2;
  if (d.memAddressReserve(&vt->base, slot_bytes * size_t(n_slots), align, 0, 0) != CUDA_SUCCESS) {
    delete vt;
    return ELLM_ERR_CUDA;
  }
  vt->handles.assign(size_t(n_slots), 0);
  vt->mapped.assign(size_t(n_slots), 0);
  vt->owned.assign(size_t(n_slots), 0);
  *out = vt;
  return ELLM_OK;
}

// cuMemCreate + cuMemMap + cuMemSetAccess for each slot (P:309 on-demand mapping; P:350 remap).
int ellm_vtensor_map(ellm_vtensor* vt, int64_t first, int64_t n) {
  if (!vt || n < 0) return ELLM_ERR_INVALID_ARG;
  if (first < 0 || first + n > vt->n_slots) return ELLM_ERR_OUT_OF_RANGE;
  for (int64_t i = first; i < first + n; ++i)
    if (vt->mapped[size_t(i)]) return ELLM_ERR_ALREADY_MAPPED;
  const Driver& d = driver();
  CUmemAllocationProp p = device_prop(vt->device);
  CUmemAccessDesc acc;
  std::memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = vt->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  int64_t t0 = now_ns();
  auto undo = [&](int64_t upto) {  // roll back slots [first, upto) on a driver failure
    for (int64_t i = first; i < upto; ++i) {
      d.memUnmap(vt->base + CUdeviceptr(i) * vt->slot_bytes, vt->slot_bytes);
      d.memRelease(vt->handles[size_t(i)]);
      vt->handles[size_t(i)] = 0;
    }
  };
  for (int64_t i = first; i < first + n; ++i) {
    CUmemGenericAllocationHandle h;
    CUdeviceptr va = vt->base + CUdeviceptr(i) * vt->slot_bytes;
    if (d.memCreate(&h, vt->slot_bytes, &p, 0) != CUDA_SUCCESS) {
      undo(i);
      return ELLM_ERR_CUDA;
    }
    if (d.memMap(va, vt->slot_bytes, 0, h, 0) != CUDA_SUCCESS) {
      d.memRelease(h);
      undo(i);
      return ELLM_ERR_CUDA;
    }
    vt->handles[size_t(i)] = h;
  }
  // one access grant for the whole contiguous run (cuMemSetAccess is required after mapping)
  if (n > 0 && d.memSetAccess(vt->base + CUdeviceptr(first) * vt->slot_bytes, vt->slot_bytes * size_t(n),
                              &acc, 1) != CUDA_SUCCESS) {
    undo(first + n);
    return ELLM_ERR_CUDA;
  }
  for (int64_t i = first; i < first + n; ++i) vt->mapped[size_t(i)] = vt->owned[size_t(i)] = 1;
  vt->n_map += n;
  vt->map_ns += now_ns() - t0;
  return ELLM_OK;
}

// cuMemUnmap + cuMemRelease ("identifies and unmaps physical memory chunks").
int ellm_vtensor_unmap(ellm_vtensor* vt, int64_t first, int64_t n) {
  if (!vt || n < 0) return ELLM_ERR_INVALID_ARG;
  if (first < 0 || first + n > vt->n_slots) return ELLM_ERR_OUT_OF_RANGE;
  for (int64_t i = first; i < first + n; ++i)
    if (!vt->mapped[size_t(i)]) return ELLM_ERR_NOT_MAPPED;
  if (n == 0) return ELLM_OK;
  if (cudaSetDevice(vt->device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return ELLM_ERR_CUDA;
  const Driver& d = driver();
  int64_t t0 = now_ns();
  for (int64_t i = first; i < first + n; ++i) {
    CUdeviceptr va = vt->base + CUdeviceptr(i) * vt->slot_bytes;
    if (d.memUnmap(va, vt->slot_bytes) != CUDA_SUCCESS) return ELLM_ERR_CUDA;
    if (vt->owned[size_t(i)] && d.memRelease(vt->handles[size_t(i)]) != CUDA_SUCCESS) return ELLM_ERR_CUDA;
    vt->handles[size_t(i)] = 0;
    vt->mapped[size_t(i)] = vt->owned[size_t(i)] = 0;
    ++vt->n_unmap;
  }
  vt->unmap_ns += now_ns() - t0;
  return ELLM_OK;
}

}  // extern "C"

namespace ellm {

// Unmap one slot without synchronising the device (the caller guarantees no pending work can
// touch it); its physical handle is released only if this slot still owns it.
int vt_unmap_slot_nosync(ellm_vtensor* vt, int64_t slot) {
  if (!vt->mapped[size_t(slot)]) return ELLM_ERR_NOT_MAPPED;
  const Driver& d = driver();
  int64_t t0 = now_ns();
  if (d.memUnmap(vt->base + CUdeviceptr(slot) * vt->slot_bytes, vt->slot_bytes) != CUDA_SUCCESS)
    return ELLM_ERR_CUDA;
  if (vt->owned[size_t(slot)] && d.memRelease(vt->handles[size_t(slot)]) != CUDA_SUCCESS) return ELLM_ERR_CUDA;
  vt->handles[size_t(slot)] = 0;
  vt->mapped[size_t(slot)] = vt->owned[size_t(slot)] = 0;
  ++vt->n_unmap;
  vt->unmap_ns += now_ns() - t0;
  return ELLM_OK;
}

// Multi-mapping: map the physical handle behind slot `src` also at slot `dst` and move
// its ownership to dst; src keeps a VA mapping of the same memory until it is unmapped (async).
int vt_map_from(ellm_vtensor* vt, int64_t dst, int64_t src) {
  if (vt->mapped[size_t(dst)]) return ELLM_ERR_ALREADY_MAPPED;
  if (!vt->mapped[size_t(src)] || !vt->owned[size_t(src)]) return ELLM_ERR_NOT_MAPPED;
  const Driver& d = driver();
  int64_t t0 = now_ns();
  const CUdeviceptr va = vt->base + CUdeviceptr(dst) * vt->slot_bytes;
  if (d.memMap(va, vt->slot_bytes, 0, vt->handles[size_t(src)], 0) != CUDA_SUCCESS) return ELLM_ERR_CUDA;
  CUmemAccessDesc acc;
  std::memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = vt->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (d.memSetAccess(va, vt->slot_bytes, &acc, 1) != CUDA_SUCCESS) {
    d.memUnmap(va, vt->slot_bytes);
    return ELLM_ERR_CUDA;
  }
  vt->handles[size_t(dst)] = vt->handles[size_t(src)];
  vt->mapped[size_t(dst)] = vt->owned[size_t(dst)] = 1;
  vt->owned[size_t(src)] = 0;
  ++vt->n_map;
  vt->map_ns += now_ns() - t0;
  return ELLM_OK;
}

}  // namespace ellm

extern "C" {

int ellm_vtensor_is_mapped(const ellm_vtensor* vt, int64_t slot) {
  if (!vt) return ELLM_ERR_INVALID_ARG;
  if (slot < 0 || slot >= vt->n_slots) return ELLM_ERR_OUT_OF_RANGE;
  return vt->mapped[size_t(slot)] ? 1 : 0;
}

void* ellm_vtensor_base(const ellm_vtensor* vt) {
  return vt ? reinterpret_cast<void*>(vt->base) : nullptr;
}

int ellm_vtensor_destroy(ellm_vtensor* vt) {
  if (!vt) return ELLM_ERR_INVALID_ARG;
  bool any = false;
  for (uint8_t m : vt->mapped) any |= bool(m);
  if (any) {
    cudaSetDevice(vt->device);
    cudaDeviceSynchronize();
  }
  const Driver& d = driver();
  for (int64_t i = 0; i < vt->n_slots; ++i)
    if (vt->mapped[size_t(i)]) {
      d.memUnmap(vt->base + CUdeviceptr(i) * vt->slot_bytes, vt->slot_bytes);
      if (vt->owned[size_t(i)]) d.memRelease(vt->handles[size_t(i)]);
    }
  if (vt->base) d.memAddressFree(vt->base, vt->slot_bytes * size_t(vt->n_slots));
  delete vt;
  return ELLM_OK;
}

}  // extern "C"

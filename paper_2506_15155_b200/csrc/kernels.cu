// kernels.cu — sm_100a kernels for the byte-moving rows of the hot path:
//   table_scatter   device mirror of the chunk tables (a2)
//   kv_append       scatter new K/V rows into chunk slabs through the table (a3)
//   chunk_copy      whole-chunk copies for deflate / inflate / migrate (a6-a8)
// All three are HBM- (or host-link-) bound byte copies: 16-byte vector accesses, several
// independent loads in flight per thread before the stores, grids sized to the SM count.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include "internal.h"

namespace ellm {
namespace {

__global__ void table_scatter_kernel(int32_t* __restrict__ table, const TableUpdate* __restrict__ up,
                                     int32_t n) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    TableUpdate u = up[i];
    table[u.index] = u.value;
  }
}

// One warp per new token row: the request / position / chunk of the row are resolved once
// (binary search over cum_rows, one table read), then the row's K and V (Hkv*d*2 bytes each,
// contiguous in k_new / v_new) move as 16-byte units, all loads in flight before the stores.
// Each (kv, head) lands as one contiguous d*2-byte row of its slab (layout [L][2][Hkv][T][d]).
constexpr int kAppendMaxPerLane = 8;  // 16-byte units per lane per kv: Hkv*d/8 <= 256
__global__ void __launch_bounds__(256) kv_append_kernel(
    const int32_t* __restrict__ req, const int32_t* __restrict__ pos0,
    const int32_t* __restrict__ cum_rows, int32_t n, int64_t total_rows, const int32_t* __restrict__ table,
    int32_t table_stride, uint8_t* __restrict__ pool, int64_t chunk_bytes, int32_t T, int32_t layer,
    int32_t Hkv, int32_t parts, const uint4* __restrict__ k_new, const uint4* __restrict__ v_new, int32_t rot) {
  const int lane = threadIdx.x & 31;
  const int units = Hkv * parts;  // 16-byte units per row and kv
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < total_rows;
       row += warps) {
    int lo = 0, hi = n - 1;  // request of this row: largest i with cum_rows[i] <= row
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(cum_rows + mid) <= row) lo = mid; else hi = mid - 1;
    }
    const int32_t p = __ldg(pos0 + lo) + int32_t(row - __ldg(cum_rows + lo));
    const int32_t c = __ldg(table + int64_t(__ldg(req + lo)) * table_stride + p / T);
    uint8_t* kdst =
        pool + int64_t(c) * chunk_bytes + (int64_t(slab_slot(c, layer, rot) * 2) * Hkv * T + (p % T)) * parts * 16;
    uint8_t* vdst = kdst + int64_t(Hkv) * T * parts * 16;
    const uint4* ksrc = k_new + row * units;
    const uint4* vsrc = v_new + row * units;
    uint4 kv_[2 * kAppendMaxPerLane];
#pragma unroll
    for (int i = 0; i < kAppendMaxPerLane; ++i) {
      const int u = lane + 32 * i;
      if (u < units) {
        kv_[i] = __ldg(ksrc + u);
        kv_[kAppendMaxPerLane + i] = __ldg(vsrc + u);
      }
    }
#pragma unroll
    for (int i = 0; i < kAppendMaxPerLane; ++i) {
      const int u = lane + 32 * i;
      if (u < units) {
        const int h = u / parts, part = u - h * parts;
        const int64_t off = (int64_t(h) * T * parts + part) * 16;
        *reinterpret_cast<uint4*>(kdst + off) = kv_[i];
        *reinterpret_cast<uint4*>(vdst + off) = kv_[kAppendMaxPerLane + i];
      }
    }
  }
}

// Chunk copy of bytes [seg_off, seg_off + seg_bytes) of each listed chunk (the whole chunk for
// swap / migrate, one layer's slabs for layer-wise offload). A warp moves one 4 KiB unit per
// iteration with 8 x 16 B loads in flight per lane before its stores (latency hiding for HBM
// and for host memory over PCIe).
constexpr int kCopyUnit = 4096;
constexpr int kCopyGrab = 16;  // units (64 KiB) a warp claims per atomic
__global__ void __launch_bounds__(256) chunk_copy_kernel(uint8_t* __restrict__ dst_base,
                                                         const int32_t* __restrict__ dst_idx,
                                                         const uint8_t* __restrict__ src_base,
                                                         const int32_t* __restrict__ src_idx,
                                                         int32_t n, int64_t chunk_bytes, int64_t seg_off,
                                                         int64_t seg_bytes, uint32_t* __restrict__ work,
                                                         int32_t rot, int64_t slab, bool src_dev, bool dst_dev) {
  // Work is claimed dynamically (one atomic per 64 KiB) rather than by a static grid stride: a
  // swap usually runs beside the persistent attention kernel, which leaves room for one copy
  // CTA per SM, so with a static split the CTAs that only become resident after the first
  // wave did their share serially at the end (measured beside C2 decode: 30 GB/s static vs
  // 52 GB/s claimed, the isolated rate).
  const int lane = threadIdx.x & 31;
  const int64_t units_per_chunk = seg_bytes / kCopyUnit;
  const int64_t total = int64_t(n) * units_per_chunk;
  for (;;) {
    uint32_t g = 0;
    if (lane == 0) g = atomicAdd(work, 1u);
    g = __shfl_sync(0xffffffffu, g, 0);
    const int64_t u0 = int64_t(g) * kCopyGrab;
    if (u0 >= total) break;
    const int64_t u1 = u0 + kCopyGrab < total ? u0 + kCopyGrab : total;
    for (int64_t w = u0; w < u1; ++w) {
      const int64_t i = w / units_per_chunk;
      const int64_t off = seg_off + (w % units_per_chunk) * kCopyUnit;  // canonical offset
      const int64_t cs = __ldg(src_idx + i), cd = __ldg(dst_idx + i);
      int64_t soff = off, doff = off;
      if (rot) {  // a pool side holds layer l's slab in slot slab_slot(c, l)
        const int32_t l = int32_t(off / slab);
        const int64_t in = off - int64_t(l) * slab;
        if (src_dev) soff = int64_t(slab_slot(cs, l, rot)) * slab + in;
        if (dst_dev) doff = int64_t(slab_slot(cd, l, rot)) * slab + in;
      }
      const uint4* s = reinterpret_cast<const uint4*>(src_base + cs * chunk_bytes + soff);
      uint4* d = reinterpret_cast<uint4*>(dst_base + cd * chunk_bytes + doff);
      uint4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcs(s + k * 32 + lane);
#pragma unroll
      for (int k = 0; k < 8; ++k) __stcs(d + k * 32 + lane, v[k]);
    }
  }
}

// D2D chunk copy (migrate, a8) through the TMA engine: one CTA per SM, one issuing thread.
// Units of kBulkUnit bytes go global -> shared (cp.async.bulk, mbarrier completion) into a ring of
// kBulkStages slots and shared -> global (cp.async.bulk store, bulk-group completion); a slot is
// reloaded as soon as the store issued kBulkLag iterations earlier has finished reading it, so
// ~kBulkStages units (~176 KiB) per SM are in flight with no register staging. Work is claimed
// kBulkGrab units per atomic, the next grab fetched before the current one is streamed.
constexpr int kBulkUnit = 16384;
constexpr int kBulkStages = 11;
constexpr int kBulkLag = 2;
constexpr int kBulkGrab = 4;
constexpr int kBulkSmem = kBulkStages * kBulkUnit + 1024;
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__global__ void __launch_bounds__(32, 1) chunk_copy_bulk_kernel(uint8_t* __restrict__ dst_base,
                                                                const int32_t* __restrict__ dst_idx,
                                                                const uint8_t* __restrict__ src_base,
                                                                const int32_t* __restrict__ src_idx,
                                                                int32_t n, int64_t chunk_bytes,
                                                                uint32_t* __restrict__ work, int32_t rot,
                                                                int64_t slab) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ alignas(8) uint64_t full[kBulkStages];
  if (threadIdx.x != 0) return;
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const uint32_t sbuf = smem_addr(buf);
  for (int s = 0; s < kBulkStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t upc = chunk_bytes / kBulkUnit;
  const int64_t total = int64_t(n) * upc;
  int64_t cur = 0, end = 0;                          // current grab [cur, end)
  uint32_t next_g = atomicAdd(work, 1u);             // the following grab, claimed ahead
  auto next_unit = [&]() -> int64_t {
    if (cur >= end) {
      cur = int64_t(next_g) * kBulkGrab;
      if (cur >= total) return -1;
      end = cur + kBulkGrab < total ? cur + kBulkGrab : total;
      next_g = atomicAdd(work, 1u);
    }
    return cur++;
  };
  auto addr = [&](int64_t w, bool dst) -> uint8_t* {
    const int64_t i = w / upc, off = (w % upc) * int64_t(kBulkUnit);  // canonical offset
    const int64_t c = __ldg((dst ? dst_idx : src_idx) + i);
    int64_t o = off;
    if (rot) {
      const int32_t l = int32_t(off / slab);
      o = int64_t(slab_slot(c, l, rot)) * slab + (off - int64_t(l) * slab);
    }
    return (dst ? dst_base : const_cast<uint8_t*>(src_base)) + c * chunk_bytes + o;
  };
  uint8_t* dptr[kBulkStages];
  int64_t nload = 0, nstore = 0;
  bool more = true;
  auto issue_load = [&]() {
    const int64_t w = next_unit();
    if (w < 0) {
      more = false;
      return;
    }
    const int st = int(nload % kBulkStages);
    const uint32_t bar = smem_addr(&full[st]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kBulkUnit) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sbuf + st * kBulkUnit), "l"(addr(w, false)), "r"(kBulkUnit), "r"(bar) : "memory");
#pragma unroll
    for (int k = 0; k < kBulkStages; ++k)
      if (k == st) dptr[k] = addr(w, true);  // select: keeps dptr[] in registers
    ++nload;
  };
  while (more && nload < kBulkStages) issue_load();
  while (nstore < nload) {
    const int st = int(nstore % kBulkStages);
    const uint32_t par = uint32_t(nstore / kBulkStages) & 1u;
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(smem_addr(&full[st])), "r"(par) : "memory");
    uint8_t* d = dptr[0];
#pragma unroll
    for (int k = 1; k < kBulkStages; ++k)
      if (k == st) d = dptr[k];
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(d), "r"(sbuf + st * kBulkUnit), "r"(kBulkUnit) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    ++nstore;
    // stores up to nstore-1-kBulkLag have read their slot: refill slots up to that one
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kBulkLag) : "memory");
    while (more && nload < nstore - kBulkLag + kBulkStages) issue_load();
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace

cudaError_t launch_table_scatter(int32_t* d_table, const TableUpdate* d_updates, int32_t n,
                                 cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int grid = std::min<int>((n + 255) / 256, 1024);
  table_scatter_kernel<<<grid, 256, 0, s>>>(d_table, d_updates, n);
  return cudaGetLastError();
}

cudaError_t launch_kv_append(const AppendDesc& d, int32_t n, int64_t total_rows, const int32_t* table,
                             int32_t table_stride, uint8_t* pool, int64_t chunk_bytes, int32_t T,
                             int32_t layer, int32_t Hkv, int32_t D, const void* k_new,
                             const void* v_new, int num_sms, cudaStream_t s, int32_t rot) {
  const int32_t parts = D / 8;
  if (Hkv * parts > 32 * kAppendMaxPerLane) return cudaErrorInvalidValue;
  const int64_t blocks = (total_rows + 7) / 8;  // 8 warps (rows) per block
  int grid = int(std::min<int64_t>(blocks, int64_t(num_sms) * 8));
  kv_append_kernel<<<grid, 256, 0, s>>>(d.req, d.pos0, d.cum_rows, n, total_rows, table, table_stride,
                                        pool, chunk_bytes, T, layer, Hkv, parts,
                                        static_cast<const uint4*>(k_new), static_cast<const uint4*>(v_new), rot);
  return cudaGetLastError();
}

cudaError_t launch_chunk_copy(uint8_t* dst_base, const int32_t* dst_idx, const uint8_t* src_base,
                              const int32_t* src_idx, int32_t n, int64_t chunk_bytes, int grid,
                              uint32_t* work, cudaStream_t s, int64_t seg_off, int64_t seg_bytes, int32_t rot,
                              int64_t slab, bool src_dev, bool dst_dev) {
  if (n <= 0) return cudaSuccess;
  if (work == nullptr) return cudaErrorInvalidValue;
  if (seg_bytes < 0) seg_bytes = chunk_bytes;
  if (seg_bytes % kCopyUnit != 0 || seg_off % 16 != 0 || seg_off + seg_bytes > chunk_bytes)
    return cudaErrorInvalidValue;
  if (rot && (slab % kCopyUnit != 0 || seg_off % kCopyUnit != 0)) return cudaErrorInvalidValue;
  // Whole-chunk D2D: the TMA bulk kernel by default when chunk_bytes is a power of two (C2's
  // 2 MiB chunks: 6534 vs 6298 GB/s device time); with 10 MiB rotated chunks the warp kernel is
  // faster (6347 vs 4615 GB/s, tools/migrate_probe.py). ELLM_D2D_BULK=1 / 0 forces either.
  const char* bulk_e = std::getenv("ELLM_D2D_BULK");
  const bool pow2 = (chunk_bytes & (chunk_bytes - 1)) == 0;
  const bool want_bulk = bulk_e ? std::atoi(bulk_e) != 0 : pow2;
  if (src_dev && dst_dev && seg_off == 0 && seg_bytes == chunk_bytes && chunk_bytes % kBulkUnit == 0 &&
      (!rot || slab % kBulkUnit == 0) && want_bulk) {
    static std::atomic<uint64_t> configured{0};  // per device (function attributes are per context)
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
      cudaError_t e = cudaFuncSetAttribute(chunk_copy_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kBulkSmem);
      if (e != cudaSuccess) return e;
      configured.fetch_or(bit, std::memory_order_release);
    }
    const int64_t bunits = int64_t(n) * (chunk_bytes / kBulkUnit);
    const int64_t bneed = (bunits + kBulkGrab - 1) / kBulkGrab;
    const int bgrid = int(std::max<int64_t>(1, std::min<int64_t>(grid / 2, bneed)));  // grid = 2 x #SM
    chunk_copy_bulk_kernel<<<bgrid, 32, kBulkSmem, s>>>(dst_base, dst_idx, src_base, src_idx, n, chunk_bytes,
                                                       work, rot, slab);
    return cudaGetLastError();
  }
  int64_t units = int64_t(n) * (seg_bytes / kCopyUnit);
  int64_t need = (units + 8 * kCopyGrab - 1) / (8 * kCopyGrab);  // one grab per warp at least
  grid = int(std::max<int64_t>(1, std::min<int64_t>(grid, need)));
  chunk_copy_kernel<<<grid, 256, 0, s>>>(dst_base, dst_idx, src_base, src_idx, n, chunk_bytes, seg_off,
                                         seg_bytes, work, rot, slab, src_dev, dst_dev);
  return cudaGetLastError();
}

// a10 consumer side: one thread waits (acquire, system scope) until this rank's gather flag has
// reached `target` — every rank's rows of the call are then in this rank's window. Bounded: after
// timeout_ns it reports and traps, so a lost peer fails the stream loudly instead of hanging it.
__global__ void gather_wait_kernel(const uint32_t* __restrict__ flag, uint32_t target, uint64_t timeout_ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (int32_t(v - target) >= 0) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      printf("ellm gather_wait: flag %u < target %u after %llu ns (peer rank missing?)\n", v, target,
             static_cast<unsigned long long>(t - t0));
      __trap();
    }
    __nanosleep(100);
  }
}

cudaError_t launch_gather_wait(const uint32_t* flag, uint32_t target, uint64_t timeout_ns, cudaStream_t s) {
  gather_wait_kernel<<<1, 1, 0, s>>>(flag, target, timeout_ns);
  return cudaGetLastError();
}

}  // namespace ellm

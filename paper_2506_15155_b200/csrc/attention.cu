// attention.cu — paged decode attention over chunk-mapped KV (SURVEY §8(a) rows a4 + a5).
//
// Computes, per request r and q-head h (kv-head g = h / group, R6):
//     o = sum_j softmax_j(scale * q.k_j) v_j,  j < len_r,
// reading k_j, v_j through the request's chunk table (P:109-112 exact attention; the
// KV eTensor's logical->physical chunk map P:307-309, read as a table, R3).
//
// B200 design:
//  * Persistent CTAs, one per SM. The flattened work space is (virtual request, stage tile);
//    CTA b owns tiles [b*W/G, (b+1)*W/G), so every SM streams the same number of bytes
//    whatever the length mix (split-K with balanced, contiguous ranges).
//  * A stage = TT tokens x HB kv-heads x {K,V} = 64 KiB (d=128). One producer warp walks the
//    chunk table and issues one 5-D TMA (cp.async.bulk.tensor, SWIZZLE_128B) per chunk piece
//    into a 3-stage mbarrier ring (192 KiB in flight per SM).
//  * 8 consumer warps; warp w owns kv-head w % HB and the 16-token subtile w / HB of every
//    stage. S = Q.K^T and O += P.V run on mma.sync m16n8k16 (bf16 in, fp32 accumulate) with
//    q-heads on the M rows. The head-dim and token orders inside a tile are permuted
//    (both sides of each dot product identically) so every smem read is one conflict-free
//    LDS.128 under the 128B swizzle and P feeds the PV MMA straight from the S accumulator.
//  * Online softmax in base 2 (exp2 of log2e-prescaled logits), row max over 4 lanes by
//    xor-shuffles, rescale skipped warp-uniformly when no row max grew.
//  * Each warp writes an fp32 partial (m, l, o) per (CTA, request); the last CTA to finish a
//    request (per-request arrival counter) merges its partials with the log-sum-exp rule and
//    writes the bf16 output, so one launch does rows a4 and a5.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cuda_bf16.h>

#include "internal.h"

namespace ellm {
namespace {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;

__host__ __device__ constexpr int stages_for(int D) { return D == 128 ? 3 : 6; }
__host__ __device__ constexpr int stage_bytes_for(int D) { return 2 * 128 * D * 2; }  // HB*TT = 128
constexpr int kQSlots = 2;  // Q ring: one slot per in-flight (owner, request) segment
constexpr int kL2PrefetchTiles = 6;  // default of Params::l2pf (set from measurements)
__host__ __device__ constexpr int q_slot_bytes_for(int D) { return 8 * 8 * D * 2; }  // HB*group <= 64 rows
__host__ __device__ constexpr int smem_bytes_for(int D) {
  return stages_for(D) * stage_bytes_for(D) + kQSlots * q_slot_bytes_for(D) + 1024 /*align*/ +
         8 * (2 * stages_for(D) + 2 * kQSlots);
}

// token permutation inside a 16-token subtile: column c of the S tile holds
// token perm16(c). perm8 = 0,5,1,4,2,7,3,6 makes the K and V smem reads bank-conflict free.
__device__ __forceinline__ int perm8(int c) { return (c & 1) ? (4 + ((c >> 1) ^ 1)) : (c >> 1); }
__device__ __forceinline__ int perm16(int c) { return (c & 8) | perm8(c & 7); }

// 16-byte block (of a d-row) that lane-quad q reads at K instruction i.
template <int D>
__device__ __forceinline__ int kblock(int q, int i) {
  if constexpr (D == 128) {
    return ((i >> 1) << 3) | (((q >> 1) << 2) | (q & 1) | ((i & 1) << 1));
  } else {
    return q + 4 * i;
  }
}
// 16-byte block of V that lane-group g reads for PV block k.
template <int D>
__device__ __forceinline__ int vblock(int g, int k) {
  if constexpr (D == 128) return g + 8 * k;
  else return 4 * (g & 1) + (g >> 1);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
// L2-only prefetch of one TMA box (no shared-memory destination, no completion)
__device__ __forceinline__ void tma_prefetch_5d(const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, int c4, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar),
      "l"(policy)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  // rows 8..15 of A (q-heads 8..15 of a group) are unused: group <= 8 (pool_create)
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct Params {
  const int32_t* table;
  const int32_t* req;
  const int32_t* len;
  const int32_t* cum_s;    // [n_vr + 1] prefix of static tiles per virtual request
  const int32_t* cum_d;    // [n_vr + 1] prefix of dynamic tiles per virtual request
  const int32_t* b_first;  // static owners of vr: CTAs [b_first, b_last] (empty if b_last < b_first)
  const int32_t* b_last;
  const int32_t* u_first;  // dynamic owners of vr: units [u_first, u_last] (empty if u_last < u_first)
  const int32_t* u_last;
  int32_t* arrivals;       // per virtual request, zero between launches
  unsigned long long* ticket;  // dynamic-unit ticket counter (monotone across launches)
  unsigned long long ticket_base;
  const int4* dyn_info;        // per unit: {vr, tile in vr, first-segment tiles, len}, {req, 0, 0, 0}
  const int32_t* dyn_ent;      // per unit: [U][npieces] chunk ids of its tiles (-1: none)
  const int4* cta_first;       // per CTA: {vr, cum_s[vr], cum_s[vr+1], len}, {req, 0, 0, 0} of its first segment
  const __nv_bfloat16* q;
  __nv_bfloat16* out;
  const uint4* k_new;      // fused decode append: [n][Hkv][d] new token rows, or nullptr
  const uint4* v_new;
  uint8_t* pool;           // pool VA base (chunk c at pool + c * chunk_bytes)
  int64_t chunk_bytes;
  int32_t Hkv;             // local kv-heads (chunk layout [L][2][Hkv][T][d])
  float* part;
  float* part_ml;
  int64_t W_s, W_d, U, n_dyn;  // static tiles; dynamic tiles; tiles per dynamic unit; units
  int32_t rec_dyn;           // record owner id of dynamic unit 0 (= G + n_vr)
  int32_t table_stride, n_vr, HG, G, T, L, layer, group, Hq;
  int32_t rot;               // slab rotation (internal.h slab_slot)
  float scale_log2;
  // a10 fused head gather (n_peer > 0; ellm_attention_gather): each merged output row is stored
  // into EVERY rank's gather window over peer memory (NVLink P2P), at global q-head
  // q_off + local head of a [n, Hq_out, D] layout, instead of into `out`; the launch's last CTA to
  // finish then adds the launch's n_vr to every rank's flag word (release, system scope).
  __nv_bfloat16* gout[kMaxPeers];
  uint32_t* gflag[kMaxPeers];
  int32_t n_peer, Hq_out, q_off;
  // a10 folded wait (ellm_gather_wait_next): the previous layer's gather must be complete in
  // this rank's window before this launch stages Q or writes (Q of layer l+1 is computed from
  // the gathered rows of layer l in a model); nullptr = no wait
  const uint32_t* wait_flag;
  uint32_t wait_target;
  unsigned long long wait_timeout_ns;
  int32_t gscope_gpu;  // 1: gather release at gpu scope (measurement knob, single-device windows only)
  uint32_t* gdone;     // gather launches: CTAs finished (monotone counter) and this launch's final value
  uint32_t gdone_target;
  unsigned long long* trace;  // ellm_set_attn_trace: [G][8] %globaltimer stamps of this launch, or null
  uint32_t range_shift;       // measurement knob: CTA i streams static range (i + shift) % G
  int32_t l2pf;               // PDL / folded wait: tiles after the first NST prefetched into L2 before waiting
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int kFirst = 1, kLast = 2, kDone = 4;  // stage metadata flags

// LSE merge of the partial records of virtual request vr, run by warps
// [w0, w0 + nw) of the last CTA to finish it:
//   M = max_p m_p,  L = sum_p 2^(m_p - M) l_p,  o = sum_p 2^(m_p - M) o_p / L   -> bf16 (RNE).
// TPR = D / (4 VEC) lanes own one q-head row, VEC float4 of o each (VEC grows with the row count
// so that more rows of the request are in flight at once: 8 rows -> VEC 1 ... 32+ rows -> VEC 4;
// measured at C4, 64 rows: 12.6 us with one row per warp pass). In one pass over the records (in
// chunks of TPR): lane k of a row loads record k's (m, l); the chunk max, the weights (broadcast by
// shuffle) and the o rows follow, DEPTH records' VEC float4 loads in flight per lane; a later chunk
// with a larger max rescales what is accumulated. Records written by other SMs are read through L2
// (__ldcg): L1 is not coherent across SMs.
template <int D, int VEC, int DEPTH>  // DEPTH: records per load batch (DEPTH x VEC float4 per lane)
__device__ __forceinline__ void merge_rows(const Params& p, int vr, int rows, int HB, int w0, int nw) {
  constexpr int TPR = D / 4 / VEC;   // lanes per row
  constexpr int RPW = 32 / TPR;      // rows per warp pass
  // record ranges: static owners (CTAs b), then dynamic owners (units u); record id of
  // (owner, vr) is owner + vr (one record per q-head row: subtile partials are combined in-CTA)
  const int64_t s0 = int64_t(__ldg(p.b_first + vr) + vr);
  const int64_t ns = int64_t(__ldg(p.b_last + vr) - __ldg(p.b_first + vr) + 1);
  const int64_t d0 = int64_t(p.rec_dyn + __ldg(p.u_first + vr) + vr);
  const int64_t nd = int64_t(__ldg(p.u_last + vr) - __ldg(p.u_first + vr) + 1);  // 0 if none
  const int64_t P = ns + nd;
  auto pid = [&](int64_t k) { return k < ns ? s0 + k : d0 + (k - ns); };
  const int ireq = vr / p.HG, hg = vr % p.HG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e4 = lane % TPR, sub = lane / TPR;
  const unsigned seg_mask = RPW == 1 ? 0xffffffffu : (((1u << TPR) - 1u) << (TPR * sub));
  for (int row0 = (warp - w0) * RPW; row0 < rows; row0 += nw * RPW) {
    const int row = row0 + sub;
    const bool live = row < rows;
    float M = -INFINITY, L = 0.f;
    float4 acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t base = 0; base < P; base += TPR) {
      const int64_t mk = base + e4;
      float2 ml = make_float2(-INFINITY, 0.f);
      if (live && mk < P) ml = __ldcg(reinterpret_cast<const float2*>(p.part_ml + (pid(mk) * rows + row) * 2));
      float cm = ml.x;
#pragma unroll
      for (int o = TPR / 2; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(seg_mask, cm, o));
      const float Mn = fmaxf(M, cm);
      if (Mn > M && M != -INFINITY) {  // a later chunk raised the max: rescale (segment-uniform)
        const float sc = ex2(M - Mn);
        L *= sc;
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          acc[v].x *= sc;
          acc[v].y *= sc;
          acc[v].z *= sc;
          acc[v].w *= sc;
        }
      }
      M = Mn;
      // a record with no valid token has m = -inf -> weight 0 (and so does every lane past P)
      const float my_w = (M == -INFINITY || ml.x == -INFINITY) ? 0.f : ex2(ml.x - M);
      L += my_w * ml.y;
      const int cnt = int(min(int64_t(TPR), P - base));
      for (int j0 = 0; j0 < cnt; j0 += DEPTH) {
        float4 ov[DEPTH][VEC];
        float wv[DEPTH];
#pragma unroll
        for (int jj = 0; jj < DEPTH; ++jj) {
          const int j = j0 + jj;
          wv[jj] = __shfl_sync(seg_mask, my_w, j % TPR, TPR);  // 0 for lanes past P
          const float4* rec = reinterpret_cast<const float4*>(p.part + (pid(base + j) * rows + row) * D);
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            ov[jj][v] = (live && j < cnt) ? __ldcg(rec + e4 + TPR * v) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int jj = 0; jj < DEPTH; ++jj) {
          const float w = (j0 + jj < cnt) ? wv[jj] : 0.f;
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            acc[v].x += w * ov[jj][v].x;
            acc[v].y += w * ov[jj][v].y;
            acc[v].z += w * ov[jj][v].z;
            acc[v].w += w * ov[jj][v].w;
          }
        }
      }
    }
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) L += __shfl_xor_sync(seg_mask, L, o);
    if (live) {
      const float inv = 1.f / L;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(acc[v].x * inv, acc[v].y * inv);
        __nv_bfloat162 hi = __floats2bfloat162_rn(acc[v].z * inv, acc[v].w * inv);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        const int col = 4 * (e4 + TPR * v);
        if (p.n_peer == 0) {
          *reinterpret_cast<uint2*>(p.out + (int64_t(ireq) * p.Hq + hg * HB * p.group + row) * D + col) = u;
        } else {  // a10: the row goes to every rank's window (own window included)
          const int64_t off = (int64_t(ireq) * p.Hq_out + p.q_off + hg * HB * p.group + row) * D + col;
          for (int i = 0; i < p.n_peer; ++i) *reinterpret_cast<uint2*>(p.gout[i] + off) = u;
        }
      }
    }
  }
}
// End-of-CTA merges: one instantiation per kernel (a runtime choice among several inlined variants
// raised the streaming loop's register pressure into spills), VEC sized for the largest row count
// the head block can have (rows = HB * group <= 8 HB): HB = 1 -> VEC 1, HB = 2 -> 2, HB >= 4 -> 4
// (C2: 32 rows in one pass of 256 lanes; the 70B shape's 64 rows in two). The merge warp 0 runs
// mid-stream when its deferred list is full is the lean DEPTH-1 form (it sits inside the
// streaming loop: a wider one there pushed the loop into spills, 25% slower launches at C2).
template <int D, int HB>
__device__ __forceinline__ void merge_request(const Params& p, int vr, int rows, int w0, int nw) {
  constexpr int VEC = D == 64 ? (HB >= 2 ? 2 : 1) : (HB >= 4 ? 4 : HB);
  merge_rows<D, VEC, 8 / VEC>(p, vr, rows, HB, w0, nw);
}
template <int D>
__device__ __forceinline__ void merge_request_lean(const Params& p, int vr, int rows, int HB) {
  merge_rows<D, 1, 1>(p, vr, rows, HB, 0, 1);
}

// One thread spins (acquire, system scope) until *flag - target >= 0 (wrapping counters);
// bounded: after timeout_ns it reports and traps so a lost peer fails the stream loudly.
__device__ __noinline__ void gather_flag_spin(const uint32_t* flag, uint32_t target,
                                              unsigned long long timeout_ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (int32_t(v - target) >= 0) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      printf("ellm attention: folded gather wait, flag %u < target %u after %llu ns\n", v, target,
             static_cast<unsigned long long>(t - t0));
      __trap();
    }
    __nanosleep(64);
  }
}

template <int D, int HB>
__global__ void __launch_bounds__(kThreads, 1)
    paged_attn_kernel(const __grid_constant__ CUtensorMap tmap, const Params p) {
  constexpr int TT = 128 / HB;          // stage tokens
  constexpr int NSUB = TT / 16;         // subtiles per stage per head
  constexpr int NST = stages_for(D);
  constexpr int SB = stage_bytes_for(D);
  constexpr int HALVES = D / 64;
  constexpr int KI = D / 32;            // K blocks (16 B) per lane per token row
  constexpr int NB = D / 64;            // V blocks per lane
  constexpr int NT = D / 8;             // PV n-tiles

  constexpr int QB = q_slot_bytes_for(D);
  constexpr int kMaxMerges = 64;        // deferred merges per CTA (the list is flushed when full)

  extern __shared__ uint8_t smem_raw[];
  __shared__ int4 s_meta[NST];          // per stage: {vr, tile within vr, record owner, flags | qslot}
  __shared__ int s_merge[kMaxMerges];   // requests this CTA completed last (merged at the end)
  __shared__ int s_n_merge;
  __shared__ int s_n_now;               // requests warp 0 merged immediately (list was full)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * SB + kQSlots * QB);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t qbase = sbase + NST * SB;  // Q ring: kQSlots x QB bytes
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + NST);
  const uint32_t qfull0 = smem_u32(bars + 2 * NST), qempty0 = smem_u32(bars + 2 * NST + kQSlots);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.trace && threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[blockIdx.x * 8 + 0] = gtimer();
    p.trace[blockIdx.x * 8 + 7] = smid;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kConsumerWarps);
    }
    for (int s = 0; s < kQSlots; ++s) {
      mbar_init(qfull0 + 8 * s, 1);
      mbar_init(qempty0 + 8 * s, kConsumerWarps);
    }
    s_n_merge = 0;
    s_n_now = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // PDL: the next attention launch on this stream may be scheduled onto SMs as this grid's
    // CTAs exit; it streams its K/V before griddepcontrol.wait and does everything that reads
    // this grid's results or writes memory after it (no-op without the launch attribute)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  __syncthreads();

  const int b = p.range_shift ? int((blockIdx.x + p.range_shift) % uint32_t(p.G)) : int(blockIdx.x);
  const int tok_box = p.T < TT ? p.T : TT;
  const int npieces = TT / tok_box;
  const int piece_bytes = 2 * HB * tok_box * D * 2;

  if (warp == kConsumerWarps) {
    // ===================== producer: work claim + table walk + TMA issue =====================
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    int stage = 0;
    uint32_t phase = 0;
    // Two tile spaces: the static space holds the first stat(vr) tiles of every request
    // (prefix cum_s), the dynamic space its last dyn(vr) tiles (prefix cum_d). This CTA streams
    // its balanced share of the static space, then dynamic U-tile units claimed from a ticket
    // counter (the next ticket is requested before the current unit is streamed, hiding the
    // atomic's latency). `owner` names the partial records a range produces: record of
    // (owner, vr) = owner + vr, unique along the monotone staircase of (owner, request) pairs.
    // the first static segment and the static range come from the host-built per-CTA record
    const int4 cf0 = __ldg(p.cta_first + 2 * b), cf1 = __ldg(p.cta_first + 2 * b + 1);
    int64_t t_begin = cf1.y, t_end = cf1.z;
    int owner = b;
    const int32_t* cum = p.cum_s;
    // Dynamic units: two tickets stay outstanding (current + next), and the next unit's
    // host-built info (first request, its tile offset / length / request id, first-segment
    // length) and chunk entries (lane t: tile t of the unit) are loaded while the current unit
    // streams, so switching units costs no dependent-load round trips.
    bool dyn = false;
    int64_t unit_start = 0;
    int4 uinfo = make_int4(0, 0, 0, 0), uinfo2 = uinfo, ninfo = uinfo, ninfo2 = uinfo;
    int32_t pent[8], npent[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) pent[k] = npent[k] = -1;
    unsigned long long tk_next = 0, tk_next2 = 0;
    if (p.n_dyn > 0 && lane == 0) {
      tk_next = atomicAdd(p.ticket, 1ull);
      tk_next2 = atomicAdd(p.ticket, 1ull);
    }
    uint32_t segc = 0;  // segments started (selects the Q slot and its parity)
    // PDL: the first segment's first NST tiles are issued before griddepcontrol.wait (the K/V of
    // this layer are not written by the previous launch: pool.cpp only sets the attribute when
    // that launch did not append into this layer); its Q is staged after the wait, before the
    // producer could block on a full ring. Fused appends (writes) also wait first.
    bool waited = false;
    int issued = 0;
    auto pdl_wait = [&]() {
      if (!waited) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (p.trace && lane == 0) p.trace[blockIdx.x * 8 + 1] = gtimer();
        if (p.wait_flag != nullptr) {  // folded a10 wait: every rank's rows of the previous layer
          if (lane == 0) gather_flag_spin(p.wait_flag, p.wait_target, p.wait_timeout_ns);
          __syncwarp();
          asm volatile("fence.proxy.async.global;" ::: "memory");  // before any TMA of Q
        }
        waited = true;
      }
    };
    bool first_static = true;
    for (;;) {
      int vr = dyn ? uinfo.x : cf0.x;
      for (int64_t tile = t_begin; tile < t_end; ++vr) {
        const bool first_dyn_seg = dyn && tile == t_begin;  // everything known from uinfo
        const bool fs = first_static;                         // everything known from cf0 / cf1
        first_static = false;
        const int64_t seg_end = first_dyn_seg ? min(t_end, t_begin + uinfo.z)
                                : fs          ? min(t_end, int64_t(cf0.z))
                                              : min(t_end, int64_t(__ldg(cum + vr + 1)));
        // a request with no tiles in this space (a short request's empty dynamic tail) is not a
        // segment: staging its Q would leave a Q slot no consumer releases
        if (seg_end <= tile) continue;
        const int ireq = vr / p.HG, hg = vr % p.HG;
        const int32_t len = first_dyn_seg ? uinfo.w : fs ? cf0.w : __ldg(p.len + ireq);
        const int32_t* trow =
            p.table + int64_t(first_dyn_seg ? uinfo2.x : fs ? cf1.x : __ldg(p.req + ireq)) * p.table_stride;
        // space coordinate of the request's first tile in this space, minus its tile offset
        const int64_t tile0 =
            first_dyn_seg ? t_begin - uinfo.y
            : fs          ? int64_t(cf0.y)
                          : __ldg(cum + vr) - (dyn ? int64_t(__ldg(p.cum_s + vr + 1) - __ldg(p.cum_s + vr)) : 0);
        const int qs = int(segc % kQSlots);
        auto stage_q = [&]() {
          if (lane == 0) {  // stage this segment's Q rows (HB*group x D, contiguous) into its slot
            mbar_wait(qempty0 + 8 * qs, ((segc / kQSlots) & 1) ^ 1);
            const uint32_t qbytes = uint32_t(HB * p.group * D * 2);
            mbar_expect_tx(qfull0 + 8 * qs, qbytes);
            bulk_load(qbase + qs * QB, p.q + (int64_t(ireq) * p.Hq + hg * HB * p.group) * D, qbytes,
                      qfull0 + 8 * qs);
          }
        };
        bool q_pending = !waited;  // first segment: Q after the first tiles and the PDL wait
        if (!q_pending) stage_q();
        for (int64_t t = tile; t < seg_end; t += 32) {
          const int cnt = int(min(int64_t(32), seg_end - t));
          int32_t ent[8];
          if (dyn) {  // prefetched: lane i of the unit holds the entries of the unit's tile i
            const int src = int(t - unit_start) + lane;
#pragma unroll
            for (int k = 0; k < 8; ++k) ent[k] = __shfl_sync(0xffffffffu, pent[k], src & 31);
          } else {
            const int64_t tokb = (t + lane - tile0) * TT;  // first position of this lane's tile
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              ent[k] = -1;
              if (k < npieces && lane < cnt && tokb + int64_t(k) * tok_box < len)
                ent[k] = __ldg(trow + (tokb + int64_t(k) * tok_box) / p.T);
            }
          }
          for (int u = 0; u < cnt; ++u) {
            int32_t e[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) e[k] = __shfl_sync(0xffffffffu, ent[k], u);
            if (q_pending && issued == NST) {  // the ring is full: Q must be on its way
              if (p.l2pf > 0 && !waited) {
                // the previous launch's slowest CTAs still run: lanes u .. u+l2pf-1 prefetch the
                // tiles after the ring's into L2 (their own entries), using the HBM bandwidth
                // its tail leaves idle; the TMA loads then hit L2 (evict-first) after the wait
                const int64_t tl = t + lane;
                if (lane >= u && lane < cnt && lane < u + p.l2pf) {
                  const int tokoff = int(((tl - tile0) * TT) % p.T);
                  const int tok_in_chunk = p.T >= TT ? tokoff : 0;
#pragma unroll
                  for (int k = 0; k < 8; ++k)
                    if (k < npieces && ent[k] >= 0)
                      tma_prefetch_5d(&tmap, 0, 0, tok_in_chunk, hg * HB,
                                      (ent[k] * p.L + slab_slot(ent[k], p.layer, p.rot)) * 2);
                }
                __syncwarp();
              }
              pdl_wait();
              stage_q();
              q_pending = false;
            }
            if (p.k_new != nullptr && (t + u - tile0 + 1) * TT >= len) {
              pdl_wait();
              // fused decode append: this is the request's last tile, which holds position
              // len-1; write the new K/V rows of heads [hg*HB, hg*HB+HB) into the chunk, then
              // order these generic-proxy stores before the tile's TMA (async proxy) read.
              const int32_t pos = len - 1;
              const int kp = int((pos - (t + u - tile0) * TT) / tok_box);  // piece holding pos
              int32_t c = e[0];
#pragma unroll
              for (int k = 1; k < 8; ++k)
                if (k == kp) c = e[k];  // select, not a dynamic index (keeps e[] in registers)
              constexpr int PARTS = D / 8, UNITS = 2 * HB * PARTS;
              for (int w = lane; w < UNITS; w += 32) {
                const int kv = w / (HB * PARTS), h = (w / PARTS) % HB, part = w % PARTS;
                const uint4* src = kv ? p.v_new : p.k_new;
                const uint4 val = __ldg(src + (int64_t(ireq) * p.Hkv + hg * HB + h) * PARTS + part);
                uint8_t* dst = p.pool + int64_t(c) * p.chunk_bytes +
                               ((int64_t(slab_slot(c, p.layer, p.rot) * 2 + kv) * p.Hkv + hg * HB + h) * p.T +
                                pos % p.T) * (D * 2) +
                               part * 16;
                *reinterpret_cast<uint4*>(dst) = val;
              }
              asm volatile("fence.proxy.async.global;" ::: "memory");
              __syncwarp();
            }
            if (lane == 0) {
              mbar_wait(empty0 + 8 * stage, phase ^ 1);
              const int64_t tl = t + u;
              s_meta[stage] = make_int4(vr, int(tl - tile0), owner + vr,
                                        (tl == tile ? kFirst : 0) | (tl == seg_end - 1 ? kLast : 0) |
                                            int((segc & 0xffff) << 8));
              int npc = 0;
#pragma unroll
              for (int k = 0; k < 8; ++k) npc += (k < npieces && e[k] >= 0);
              mbar_expect_tx(full0 + 8 * stage, uint32_t(npc * piece_bytes));
              const int tokoff = int(((tl - tile0) * TT) % p.T);
              const int tok_in_chunk = p.T >= TT ? tokoff : 0;
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (k < npieces && e[k] >= 0)
                  tma_load_5d(sbase + stage * SB + k * piece_bytes, &tmap, 0, 0, tok_in_chunk, hg * HB,
                              (e[k] * p.L + slab_slot(e[k], p.layer, p.rot)) * 2, full0 + 8 * stage, policy);
            }
            __syncwarp();
            ++issued;
            if (++stage == NST) { stage = 0; phase ^= 1; }
          }
        }
        if (q_pending) {  // a first segment of fewer than NST tiles
          pdl_wait();
          stage_q();
        }
        tile = seg_end;
        ++segc;
      }
      // next range: the unit of the next ticket (two failing tickets per CTA end the phase)
      if (p.n_dyn == 0) break;
      const int64_t u = int64_t(__shfl_sync(0xffffffffu, tk_next, 0) - p.ticket_base);
      if (u >= p.n_dyn) break;
      const int ul = p.U * npieces;  // entries per unit
      if (!dyn) {  // entering the dynamic phase: this unit's info was not prefetched
        ninfo = __ldg(p.dyn_info + 2 * u);
        ninfo2 = __ldg(p.dyn_info + 2 * u + 1);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          npent[k] = (lane < p.U && k < npieces) ? __ldg(p.dyn_ent + u * ul + lane * npieces + k) : -1;
      }
      uinfo = ninfo;
      uinfo2 = ninfo2;
#pragma unroll
      for (int k = 0; k < 8; ++k) pent[k] = npent[k];
      const int64_t u2 = int64_t(__shfl_sync(0xffffffffu, tk_next2, 0) - p.ticket_base);
      if (u2 < p.n_dyn) {  // prefetch the following unit while this one streams
        ninfo = __ldg(p.dyn_info + 2 * u2);
        ninfo2 = __ldg(p.dyn_info + 2 * u2 + 1);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          npent[k] = (lane < p.U && k < npieces) ? __ldg(p.dyn_ent + u2 * ul + lane * npieces + k) : -1;
      }
      if (lane == 0) {
        tk_next = tk_next2;
        tk_next2 = atomicAdd(p.ticket, 1ull);
      }
      dyn = true;
      t_begin = u * p.U;
      t_end = min(p.W_d, t_begin + p.U);
      unit_start = t_begin;
      owner = p.rec_dyn + int(u);
      cum = p.cum_d;
    }
    // no more work: publish DONE through the next stage (plain arrive, no bytes)
    if (lane == 0) {
      mbar_wait(empty0 + 8 * stage, phase ^ 1);
      s_meta[stage] = make_int4(0, 0, 0, kDone);
      mbar_arrive(full0 + 8 * stage);
    }
    return;
  }

  // ========================= consumers =========================
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: before any read of Q or any write
  const int hh = warp % HB, j = warp / HB;
  const int g = lane >> 2, q = lane & 3;
  // smem byte offsets (within a stage) of this lane's K and V reads; fixed for the kernel
  auto soff = [&](int kv, int tau, int blk) -> uint32_t {
    const int piece = tau / tok_box, t = tau % tok_box;
    const int line = ((kv * HB + hh) * tok_box + t) * HALVES + (blk >> 3);
    return uint32_t(piece * piece_bytes + line * 128 + (((blk & 7) ^ (line & 7)) << 4));
  };
  uint32_t koff[2][KI], voff[4][NB];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int i = 0; i < KI; ++i) koff[nt][i] = soff(0, 16 * j + perm16(nt * 8 + g), kblock<D>(q, i));
  int vcol[4] = {2 * q, 2 * q + 1, 2 * q + 8, 2 * q + 9};
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int k = 0; k < NB; ++k) voff[r][k] = soff(1, 16 * j + perm16(vcol[r]), vblock<D>(g, k));

  const int rows = HB * p.group;
  const int row = hh * p.group + g;  // q-head row within a head group
  int stage = 0;
  uint32_t phase = 0;
  uint4 qb[KI];
  float o[NT][4];
  float m_run = -INFINITY, l_run = 0.f;
  int32_t len = 0;
  bool first_data = true;
  for (;;) {
    mbar_wait(full0 + 8 * stage, phase);
    if (p.trace && threadIdx.x == 0 && first_data) p.trace[blockIdx.x * 8 + 2] = gtimer();
    first_data = false;
    const int4 meta = s_meta[stage];
    if (meta.w & kDone) break;
    const int vr = meta.x;
    if (meta.w & kFirst) {  // a new (owner, request) segment: its Q and fresh softmax state
      const int ireq = vr / p.HG;
      len = __ldg(p.len + ireq);
      const uint32_t segc = uint32_t(meta.w) >> 8;  // Q rows were staged by the producer
      const int qs = int(segc % kQSlots);
      mbar_wait(qfull0 + 8 * qs, (segc / kQSlots) & 1);
      if (g < p.group) {
        const uint32_t qrow = qbase + qs * QB + uint32_t(row * D * 2);
#pragma unroll
        for (int i = 0; i < KI; ++i) qb[i] = lds128(qrow + 16 * kblock<D>(q, i));
      } else {
#pragma unroll
        for (int i = 0; i < KI; ++i) qb[i] = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty0 + 8 * qs);
#pragma unroll
      for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
      m_run = -INFINITY;
      l_run = 0.f;
    }
    const uint32_t st = sbase + stage * SB;
    const int valid = int(min(int64_t(16), int64_t(len) - (int64_t(meta.y) * TT + 16 * j)));
    if (valid > 0) {
      // ---- S = Q K^T : rows = q-heads, cols = 16 tokens (two n-tiles) ----
      float s[2][4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
        for (int i = 0; i < KI; ++i) {
          const uint4 kk = lds128(st + koff[nt][i]);
          mma_bf16(s[nt], qb[i].x, qb[i].y, kk.x, kk.y);
          mma_bf16(s[nt], qb[i].z, qb[i].w, kk.z, kk.w);
        }
      }
      // ---- online softmax (base 2) on row g ----
      float x[2][2];
      float mx = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v = s[nt][c] * p.scale_log2;
          if (perm16(nt * 8 + 2 * q + c) >= valid) v = -INFINITY;
          x[nt][c] = v;
          mx = fmaxf(mx, v);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_run, mx);
      if (__any_sync(0xffffffffu, m_new > m_run)) {
        const float alpha = ex2(m_run - m_new);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          o[n][0] *= alpha;
          o[n][1] *= alpha;
        }
        l_run *= alpha;
        m_run = m_new;
      }
      float pr[2][2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          pr[nt][c] = ex2(x[nt][c] - m_run);
          l_run += pr[nt][c];
        }
      const uint32_t pa0 = pack_bf16(pr[0][0], pr[0][1]);
      const uint32_t pa2 = pack_bf16(pr[1][0], pr[1][1]);
      // ---- O += P V : V rows regrouped token-pairwise with byte permutes ----
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        uint4 v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) v[r] = lds128(st + voff[r][k]);
        if (valid < 16) {  // tail: never multiply garbage rows (could be Inf/NaN) by P = 0
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (perm16(vcol[r]) >= valid) v[r] = make_uint4(0, 0, 0, 0);
        }
        const uint32_t* v0 = &v[0].x;
        const uint32_t* v1 = &v[1].x;
        const uint32_t* v2 = &v[2].x;
        const uint32_t* v3 = &v[3].x;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          mma_bf16(o[8 * k + 2 * u], pa0, pa2, __byte_perm(v0[u], v1[u], 0x5410),
                   __byte_perm(v2[u], v3[u], 0x5410));
          mma_bf16(o[8 * k + 2 * u + 1], pa0, pa2, __byte_perm(v0[u], v1[u], 0x7632),
                   __byte_perm(v2[u], v3[u], 0x7632));
        }
      }
    }
    __syncwarp();
    const bool seg_last = (meta.w & kLast) != 0;
    // with NSUB > 1 subtile warps per head, a segment's last stage doubles as the scratch of the
    // in-CTA combine below: it is released only after that
    const uint32_t cur_stage = uint32_t(stage);
    if (lane == 0 && !(seg_last && NSUB > 1)) mbar_arrive(empty0 + 8 * stage);
    if (++stage == NST) { stage = 0; phase ^= 1; }
    if (!seg_last) continue;

    // ---- partial record of (owner, virtual request vr): one per q-head row ----
    float l_tot = l_run + __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 2);
    // this lane's o fragment as 16-byte pieces: piece k of the row at float offset foff(k)
    auto write_frag = [&](float* dst) {
      if constexpr (D == 128) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          float4* d4 = reinterpret_cast<float4*>(dst + 64 * h2 + 16 * q);
          d4[0] = make_float4(o[8 * h2 + 0][0], o[8 * h2 + 1][0], o[8 * h2 + 2][0], o[8 * h2 + 3][0]);
          d4[1] = make_float4(o[8 * h2 + 4][0], o[8 * h2 + 5][0], o[8 * h2 + 6][0], o[8 * h2 + 7][0]);
          d4[2] = make_float4(o[8 * h2 + 0][1], o[8 * h2 + 1][1], o[8 * h2 + 2][1], o[8 * h2 + 3][1]);
          d4[3] = make_float4(o[8 * h2 + 4][1], o[8 * h2 + 5][1], o[8 * h2 + 6][1], o[8 * h2 + 7][1]);
        }
      } else {
        float4* a = reinterpret_cast<float4*>(dst + 8 * q);
        a[0] = make_float4(o[0][0], o[1][0], o[2][0], o[3][0]);
        a[1] = make_float4(o[4][0], o[5][0], o[6][0], o[7][0]);
        float4* c = reinterpret_cast<float4*>(dst + 32 + 8 * q);
        c[0] = make_float4(o[0][1], o[1][1], o[2][1], o[3][1]);
        c[1] = make_float4(o[4][1], o[5][1], o[6][1], o[7][1]);
      }
    };
    if constexpr (NSUB == 1) {
      if (g < p.group) {
        const int64_t rec = int64_t(meta.z) * rows + row;
        write_frag(p.part + rec * D);
        if (q == 0) *reinterpret_cast<float2*>(p.part_ml + rec * 2) = make_float2(m_run, l_tot);
      }
    } else {
      // In-CTA combine of the NSUB subtile partials of each q-head row (same LSE rule as the
      // merge), so a segment leaves ONE record per row instead of NSUB: the end-of-launch merges
      // then read NSUB times fewer records (measured at the 8-way C4 shard, NSUB = 8: ~26 -> ~3
      // records per request; the merge is on the launch's critical path). Scratch: the stage
      // just consumed, [NSUB][rows][D] fp32 + [NSUB][rows] (m, l), at most 32 KiB + 512 B.
      float* scr = reinterpret_cast<float*>(smem + cur_stage * SB);
      float* scr_ml = scr + NSUB * rows * D;
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");  // every warp's K/V reads done
      if (g < p.group) {
        write_frag(scr + (j * rows + row) * D);
        if (q == 0) *reinterpret_cast<float2*>(scr_ml + (j * rows + row) * 2) = make_float2(m_run, l_tot);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
      constexpr int LPR = D / 4, RPW = 32 / LPR;
      const int e4 = lane % LPR, sub = lane / LPR;
      for (int r = warp * RPW + sub; r < rows; r += kConsumerWarps * RPW) {
        float M = -INFINITY;
#pragma unroll
        for (int jj = 0; jj < NSUB; ++jj) M = fmaxf(M, scr_ml[(jj * rows + r) * 2]);
        float L = 0.f;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int jj = 0; jj < NSUB; ++jj) {
          const float2 ml = *reinterpret_cast<const float2*>(scr_ml + (jj * rows + r) * 2);
          const float w = ml.x == -INFINITY ? 0.f : ex2(ml.x - M);  // an empty subtile: weight 0
          const float4 v = reinterpret_cast<const float4*>(scr + (jj * rows + r) * D)[e4];
          L += w * ml.y;
          acc.x += w * v.x;
          acc.y += w * v.y;
          acc.z += w * v.z;
          acc.w += w * v.w;
        }
        const int64_t rec = int64_t(meta.z) * rows + r;
        reinterpret_cast<float4*>(p.part + rec * D)[e4] = acc;
        if (e4 == 0) *reinterpret_cast<float2*>(p.part_ml + rec * 2) = make_float2(M, L);
      }
      // generic-proxy use of the stage is over before the TMA (async proxy) refills it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
      if (lane == 0) mbar_arrive(empty0 + 8 * cur_stage);
    }
    // ---- arrival: the owner that completes request vr's count merges it (a5, fused) ----
    // bar.sync orders every consumer's record stores before thread 0's gpu-scope fence +
    // atomic (fences are cumulative); only warp 0 waits for the atomic's result, and the merge
    // itself is deferred to the end of this CTA's work so segment switches stay cheap.
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
    if (warp == 0) {
      int now = 0;
      if (lane == 0) {
        __threadfence();
        const int bf = __ldg(p.b_first + vr), bl = __ldg(p.b_last + vr);
        const int uf = __ldg(p.u_first + vr), ul = __ldg(p.u_last + vr);
        const int owners = (bl >= bf ? bl - bf + 1 : 0) + (ul >= uf ? ul - uf + 1 : 0);
        const int old = atomicAdd(p.arrivals + vr, 1);
        if (old == owners - 1) {
          p.arrivals[vr] = 0;  // every owner of vr has arrived: re-arm for the next launch
          __threadfence();
          if (s_n_merge < kMaxMerges) s_merge[s_n_merge++] = vr;
          else now = 1;        // deferred list full: warp 0 merges this one right away
        }
      }
      if (__shfl_sync(0xffffffffu, now, 0)) {
        merge_request_lean<D>(p, vr, rows, HB);
        if (lane == 0) ++s_n_now;
      }
    }
  }
  // ---- end of this CTA's work: all consumer warps merge the requests it completed ----
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 8 + 3] = gtimer();
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
  __threadfence();
  for (int k = 0; k < s_n_merge; ++k)
    merge_request<D, HB>(p, s_merge[k], rows, 0, kConsumerWarps);
  if (p.trace && threadIdx.x == 0) {
    p.trace[blockIdx.x * 8 + 4] = gtimer();
    p.trace[blockIdx.x * 8 + 6] = (unsigned long long)(s_n_merge + s_n_now);
  }
  if (p.n_peer > 0) {
    // a10 signal. Every CTA orders its row stores before a gpu-scope count (the named barrier
    // gathers the consumer threads' stores at thread 0, whose acq_rel fence + relaxed add is a
    // release); the CTA whose add completes the launch's count has then observed every CTA's
    // rows, and one system-scope fence (cumulative) + a relaxed add of all n_vr merged requests
    // to every rank's flag publishes them. One membar.sys per launch instead of one per CTA
    // (measured: a membar.sys in every CTA cost ~6 us of a 50 us 8-way launch).
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
    if (threadIdx.x == 0) {
      uint32_t old;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.gdone) : "memory");
      if (old == p.gdone_target - 1u) {
        const uint32_t all = uint32_t(p.n_vr);
        if (p.gscope_gpu) {  // measurement knob (ELLM_GATHER_SCOPE=gpu): every window on this device
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          for (int i = 0; i < p.n_peer; ++i)
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p.gflag[i]), "r"(all) : "memory");
        } else {
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          for (int i = 0; i < p.n_peer; ++i)
            asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p.gflag[i]), "r"(all) : "memory");
        }
      }
    }
  }
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 8 + 5] = gtimer();
}

template <int D, int HB>
cudaError_t launch_t(const CUtensorMap& tmap, const Params& prm, int G, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes_for(D);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, paged_attn_kernel<D, HB>, tmap, prm);
}

}  // namespace

int attn_heads_per_block(int32_t Hkv) { return Hkv >= 8 ? 8 : Hkv; }
int attn_stage_tokens(int32_t HB) { return 128 / HB; }

template <int D>
static cudaError_t configure_d(int32_t HB) {
  const void* f = nullptr;
  switch (HB) {
    case 1: f = reinterpret_cast<const void*>(paged_attn_kernel<D, 1>); break;
    case 2: f = reinterpret_cast<const void*>(paged_attn_kernel<D, 2>); break;
    case 4: f = reinterpret_cast<const void*>(paged_attn_kernel<D, 4>); break;
    case 8: f = reinterpret_cast<const void*>(paged_attn_kernel<D, 8>); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes_for(D));
}

cudaError_t attn_configure(int32_t D, int32_t HB) {
  return D == 128 ? configure_d<128>(HB) : D == 64 ? configure_d<64>(HB) : cudaErrorInvalidValue;
}

// 5-D view of the pool: (64 elems, d/64 halves, T tokens, Hkv heads, chunk*L*2 + layer*2 + kv)
// with the box (64, d/64, min(T,TT), HB, 2): one TMA = K and V of HB heads for up to TT tokens.
cudaError_t encode_kv_tensor_map(CUtensorMap* map, void* pool_base, int64_t max_chunks,
                                 const AttnShape& sh) {
  const Driver& d = driver();
  if (!d.ok) return cudaErrorNotSupported;
  cuuint64_t dims[5] = {64, cuuint64_t(sh.D / 64), cuuint64_t(sh.T), cuuint64_t(sh.Hkv),
                        cuuint64_t(max_chunks) * sh.L * 2};
  cuuint64_t strides[4] = {128, cuuint64_t(sh.D) * 2, cuuint64_t(sh.T) * sh.D * 2,
                           cuuint64_t(sh.Hkv) * sh.T * sh.D * 2};
  cuuint32_t box[5] = {64, cuuint32_t(sh.D / 64), cuuint32_t(sh.T < sh.TT ? sh.T : sh.TT),
                       cuuint32_t(sh.HB), 2};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = d.tensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, pool_base, dims, strides,
                                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_paged_attention(const CUtensorMap& tmap, const AttnShape& sh, const AttnDesc& d,
                                   int32_t n, int32_t n_vr, const AttnPlan& plan,
                                   const int32_t* table, int32_t table_stride, int32_t layer,
                                   const void* q, void* out, float* part, float* part_ml,
                                   int32_t* arrivals, float scale, cudaStream_t s, int* launches) {
  (void)n;
  const int32_t G = plan.G;
  Params prm;
  prm.table = table;
  prm.req = d.req;
  prm.len = d.len;
  prm.cum_s = d.cum_s;
  prm.cum_d = d.cum_d;
  prm.b_first = d.b_first;
  prm.b_last = d.b_last;
  prm.u_first = d.u_first;
  prm.u_last = d.u_last;
  prm.arrivals = arrivals;
  prm.ticket = plan.ticket;
  prm.ticket_base = plan.ticket_base;
  prm.dyn_info = reinterpret_cast<const int4*>(plan.dyn_info);
  prm.dyn_ent = plan.dyn_ent;
  prm.cta_first = reinterpret_cast<const int4*>(plan.cta_first);
  prm.q = static_cast<const __nv_bfloat16*>(q);
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.k_new = static_cast<const uint4*>(plan.k_new);
  prm.v_new = static_cast<const uint4*>(plan.v_new);
  prm.pool = plan.pool;
  prm.chunk_bytes = plan.chunk_bytes;
  prm.Hkv = sh.Hkv;
  prm.part = part;
  prm.part_ml = part_ml;
  prm.W_s = plan.W_s;
  prm.W_d = plan.W_d;
  prm.U = plan.U;
  prm.n_dyn = plan.n_dyn;
  prm.rec_dyn = G + n_vr;
  prm.table_stride = table_stride;
  prm.n_vr = n_vr;
  prm.HG = sh.HG;
  prm.G = G;
  prm.T = sh.T;
  prm.L = sh.L;
  prm.layer = layer;
  prm.rot = sh.rot;
  prm.group = sh.group;
  prm.Hq = sh.Hq;
  prm.scale_log2 = scale * 1.4426950408889634f;
  prm.n_peer = plan.n_peer;
  prm.Hq_out = plan.Hq_out;
  prm.q_off = plan.q_off;
  for (int i = 0; i < kMaxPeers; ++i) {
    prm.gout[i] = static_cast<__nv_bfloat16*>(plan.gout[i]);
    prm.gflag[i] = plan.gflag[i];
  }
  prm.gdone = plan.gdone;
  prm.trace = plan.trace;
  prm.range_shift = plan.range_shift;
  {
    // tiles prefetched into L2 while a launch waits on its predecessor (PDL) or on the peers'
    // gather flags; ELLM_ATTN_L2PF overrides (0 = off)
    static const int l2pf = [] {
      const char* v = std::getenv("ELLM_ATTN_L2PF");
      return v ? std::max(0, std::min(31, std::atoi(v))) : kL2PrefetchTiles;
    }();
    prm.l2pf = (plan.pdl || plan.wait_flag != nullptr) ? l2pf : 0;
  }
  prm.gdone_target = plan.gdone_target;
  prm.wait_flag = plan.wait_flag;
  prm.wait_target = plan.wait_target;
  prm.wait_timeout_ns = plan.wait_timeout_ns;
  {
    const char* g = std::getenv("ELLM_GATHER_SCOPE");
    prm.gscope_gpu = (g && g[0] == 'g') ? 1 : 0;
  }
  cudaError_t e;
  if (sh.D == 128) {
    switch (sh.HB) {
      case 1: e = launch_t<128, 1>(tmap, prm, G, s, plan.pdl); break;
      case 2: e = launch_t<128, 2>(tmap, prm, G, s, plan.pdl); break;
      case 4: e = launch_t<128, 4>(tmap, prm, G, s, plan.pdl); break;
      default: e = launch_t<128, 8>(tmap, prm, G, s, plan.pdl); break;
    }
  } else {
    switch (sh.HB) {
      case 1: e = launch_t<64, 1>(tmap, prm, G, s, plan.pdl); break;
      case 2: e = launch_t<64, 2>(tmap, prm, G, s, plan.pdl); break;
      case 4: e = launch_t<64, 4>(tmap, prm, G, s, plan.pdl); break;
      default: e = launch_t<64, 8>(tmap, prm, G, s, plan.pdl); break;
    }
  }
  *launches = e == cudaSuccess ? 1 : 0;
  return e;
}

}  // namespace ellm

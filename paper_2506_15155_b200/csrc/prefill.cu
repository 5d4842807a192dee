// prefill.cu — chunked-prefill attention over chunk-mapped KV on the 5th-generation tensor cores
// ("chunked prefill"; P:109-112 causal attention over the KV cache).
//
// Computes, for the last n_q positions of each listed request (query k at position
// P = len - n_q + k) and every q-head h (kv-head g = h / group, R6):
//     o = sum_{j <= P} softmax_j(scale * q.k_j) v_j,
// reading k_j, v_j through the request's chunk table (R3).
//
// B200 design (f4):
//  * One CTA per work item = (request, kv-head, block of 128/group query positions). Its M = 128
//    MMA rows are (position, q-head of the group) pairs, so one K/V tile feeds every head of the
//    group. Items are ordered by decreasing tile count (longest first).
//  * Warp 0: TMA producer. Q once (SWIZZLE_128B, K-major rows), then per 128-key tile the
//    chunk table's pieces: one TMA box (64 d-elements x min(T,128) tokens) per (piece, K/V,
//    64-wide half of d) into a 2-stage mbarrier ring laid out [half][token][64] — the canonical
//    UMMA K-major layout for K and MN-major layout for V.
//  * Warp 1: allocates 512 TMEM columns and issues tcgen05.mma (one thread): S = Q.K^T into a
//    double-buffered fp32 TMEM tile (cols 0-127 / 128-255), then O += P.V into cols 256+
//    (P from shared memory, V MN-major), committing to mbarriers (tcgen05.commit).
//  * Warps 2-5: softmax, one thread per TMEM lane = one MMA row. tcgen05.ld of the S row, causal
//    mask, base-2 online softmax with lazy rescaling (O in TMEM is rescaled only when the row max
//    grows by more than 2^8), P written as bf16 into shared memory in the swizzled K-major layout,
//    and at the end O / l -> bf16 -> global.
#include <atomic>
#include <cstdlib>

#include <cuda_bf16.h>

#include "internal.h"

namespace ellm {
namespace {

constexpr int kM = 128;         // MMA rows per Q tile (TMEM lanes)
constexpr int kN = 128;         // keys per tile
constexpr int kQTiles = 2;      // Q tiles per CTA (ping-pong: one tile's softmax hides the other's MMAs)
constexpr int kKStages = 2;     // K ring depth
constexpr int kVStages = 2;     // V ring depth
#ifndef ELLM_PF_SPLIT
#define ELLM_PF_SPLIT 1
#endif
constexpr int kSplit = ELLM_PF_SPLIT;  // softmax warps per (Q tile, TMEM lane quarter): each owns kN / kSplit keys
constexpr int kSoftmaxWarps = 4 * kQTiles * kSplit;
constexpr int kThreads = 64 + 32 * kSoftmaxWarps;  // warp 0 TMA, warp 1 MMA, 8 softmax warps per Q tile
constexpr uint32_t kTmemCols = 512;
constexpr float kRescaleHeadroom = 8.f;
  // log2 units: P <= 2^8 before O is rescaled

template <int D>
struct Layout {
  static constexpr int TILE = kN * D * 2;   // one K or V tile: [D/64][128 tokens][64] bf16
  static constexpr int QT = kM * D * 2;     // one Q tile: [D/64][128 rows][64]
  static constexpr int off_q = 0;           // Q tile x at off_q + x*QT
  static constexpr int off_k = kQTiles * QT;                // K stage s at off_k + s*TILE
  static constexpr int off_v = off_k + kKStages * TILE;     // V stage s at off_v + s*TILE
  static constexpr int off_bar = off_v + kVStages * TILE;
  static constexpr int off_red = off_bar + 256;  // [2 parities][kQTiles][kSplit][128 rows] fp32: row-max exchange
  static constexpr int bytes = off_red + 2 * kQTiles * kSplit * kM * 4 + 1024;
  static_assert(bytes <= 232448, "shared memory per CTA");
};

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
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                       uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_5d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                       int c4, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar),
      "l"(policy)
      : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA / integer pipes (no MUFU): round-to-nearest split x = j + f, f in [-1/2, 1/2],
// 2^f by a cubic (relative-error fit on [-1/2, 1/2]: < 7.5e-5, far below bf16's 2^-9 half-ulp
// of P; the arithmetic below is emulated in numpy and checked in tests/test_prefill_exp2.py), then
// j added to the exponent field. Inputs are clamped at -125 so the result stays a normal float
// (>= 2^-125.5; masked scores, -inf, give that instead of 0 — 1e-38 of a zeroed or finite V row).
constexpr float kE2C3 = 0.05517161f, kE2C2 = 0.24261114f, kE2C1 = 0.693261f, kE2C0 = 0.99992807f;
// sm_100 packed fp32 pairs (one FFMA2 / FADD2 instead of two FFMA / FADD: fewer issue slots)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d)
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)),
        "l"(*reinterpret_cast<const uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d)
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}
// The FMA-pipe exp2 above on a pair with packed fp32 ops (FADD2 / FFMA2; x - (r - M) as an exact
// fma by -1): 12 instructions per two exponentials.
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 M = make_float2(12582912.f, 12582912.f), mM = make_float2(-12582912.f, -12582912.f);
  const float2 r = fadd2(x, M);
  const float2 f = ffma2(fadd2(r, mM), make_float2(-1.f, -1.f), x);
  float2 q = ffma2(make_float2(kE2C3, kE2C3), f, make_float2(kE2C2, kE2C2));
  q = ffma2(q, f, make_float2(kE2C1, kE2C1));
  q = ffma2(q, f, make_float2(kE2C0, kE2C0));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(r.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(r.y) << 23)));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---- tcgen05 -------------------------------------------------------------------------------
// Shared-memory matrix descriptor (sm100 "version 1"), 128-byte swizzle, 8-row atoms of
// 1024 B. K-major: rows of 64 elements, LBO unused (16 B), SBO = 1024 B between 8-row groups.
// MN-major: 64-element MN blocks `lbo` bytes apart, 8-row K groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// Instruction descriptor, kind::f16: fp32 accumulate, bf16 A and B, A K-major, B K- or MN-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(b_mn_major) << 16) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}
// tcgen05.mma / commit are single-thread instructions: the whole MMA warp runs the issue loop
// with warp-uniform operands (so they live in uniform registers) and elect.sync picks the one
// thread that issues (a lane-0-only branch made ptxas wrap every MMA in an elect / broadcast /
// R2UR loop: ~10 dependent instructions per MMA, measured as the MMA warp's critical path).
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

#define ELLM_R32(i) "=r"(r[i])
// 32 consecutive TMEM columns of this thread's lane -> registers
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : ELLM_R32(0), ELLM_R32(1), ELLM_R32(2), ELLM_R32(3), ELLM_R32(4), ELLM_R32(5), ELLM_R32(6), ELLM_R32(7),
        ELLM_R32(8), ELLM_R32(9), ELLM_R32(10), ELLM_R32(11), ELLM_R32(12), ELLM_R32(13), ELLM_R32(14),
        ELLM_R32(15), ELLM_R32(16), ELLM_R32(17), ELLM_R32(18), ELLM_R32(19), ELLM_R32(20), ELLM_R32(21),
        ELLM_R32(22), ELLM_R32(23), ELLM_R32(24), ELLM_R32(25), ELLM_R32(26), ELLM_R32(27), ELLM_R32(28),
        ELLM_R32(29), ELLM_R32(30), ELLM_R32(31)
      : "r"(taddr));
}
#undef ELLM_R32
#define ELLM_R16(i) "=r"(r[i])
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : ELLM_R16(0), ELLM_R16(1), ELLM_R16(2), ELLM_R16(3), ELLM_R16(4), ELLM_R16(5), ELLM_R16(6), ELLM_R16(7),
        ELLM_R16(8), ELLM_R16(9), ELLM_R16(10), ELLM_R16(11), ELLM_R16(12), ELLM_R16(13), ELLM_R16(14),
        ELLM_R16(15)
      : "r"(taddr));
}
#undef ELLM_R16
#define ELLM_W16(i) "r"(r[i])
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      ELLM_W16(0), ELLM_W16(1), ELLM_W16(2), ELLM_W16(3), ELLM_W16(4), ELLM_W16(5), ELLM_W16(6), ELLM_W16(7),
      ELLM_W16(8), ELLM_W16(9), ELLM_W16(10), ELLM_W16(11), ELLM_W16(12), ELLM_W16(13), ELLM_W16(14), ELLM_W16(15)
      : "memory");
}
#undef ELLM_W16
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// A operand from tensor memory (P: M=128 lanes x K keys, two bf16 per 32-bit column)
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

struct PParams {
  const int4* work;        // [n_work][2]: {req, len, q_row0, p0}, {n_valid, kvh, n_tiles, 0}
  const int32_t* table;
  __nv_bfloat16* out;      // [rows][Hq][D]
  int32_t table_stride, Hq, group, T, L, layer, Hkv;
  int32_t rot;             // slab rotation (internal.h slab_slot)
  int32_t runs;            // run maps usable (else one box per chunk through maps.kv)
  float scale_log2;
  unsigned long long* trace;  // ellm_set_attn_trace buffer: CTA 0's per-tile handoff clocks, or null
};
__device__ __forceinline__ void pf_stamp(const PParams& p, int t, int k) {
  if (p.trace != nullptr && blockIdx.x == 0 && t < 16) p.trace[t * 16 + k] = clock64();
}

// One CTA per work item = (request, kv-head, block of 2 x 128/group query positions): Q tile x
// (x = 0, 1) holds the block's x-th 128/group positions x group heads as its M = 128 rows.
// TMEM (512 columns): S_x at [128x, 128x + 128) — overwritten in place by P_x as bf16 pairs in its
// first 64 columns — and O_x at [256 + 128x, 256 + 128x + D). Both tiles share every K/V tile.
// The MMA thread issues, per key tile t:  PV_0(t), S_0(t+1), PV_1(t), S_1(t+1), so while softmax
// warpgroup x works on S_x(t+1) the tensor pipe runs the other tile's P.V and S.
// EMU: of every 8 pairs of softmax exponentials, this many run on the FMA pipe (ex2_fma2), the rest
// on MUFU
template <int D, int EMU>
__global__ void __launch_bounds__(kThreads, 1)
    prefill_kernel(const __grid_constant__ PrefillMaps maps, const PParams p) {
  using LY = Layout<D>;
  constexpr int HALVES = D / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t bar0 = sb + LY::off_bar;
  // barriers (8 B each): q_full, k_full[KS], k_empty[KS], v_full[VS], v_empty[VS],
  // s_full[2], p_full[2], o_full[2]; then the TMEM address
  const uint32_t q_full = bar0, k_full = bar0 + 8, k_empty = k_full + 8 * kKStages,
                 v_full = k_empty + 8 * kKStages, v_empty = v_full + 8 * kVStages,
                 s_full = v_empty + 8 * kVStages, p_full = s_full + 16, o_full = p_full + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + LY::off_bar + 224);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4 w0 = p.work[2 * blockIdx.x], w1 = p.work[2 * blockIdx.x + 1];
  const int req = w0.x, q_row0 = w0.z, p0 = w0.w;
  const int n_valid = w1.x, kvh = w1.y, n_tiles = w1.z;
  const int last_key = p0 + n_valid - 1;  // the block's largest query position (< len)
  const int bp = kM / p.group;             // positions per Q tile
  const int nq = n_valid > bp ? 2 : 1;     // Q tiles with any valid row

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(k_full + 8 * s, 1);
      mbar_init(k_empty + 8 * s, 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(v_full + 8 * s, 1);
      mbar_init(v_empty + 8 * s, 1);
    }
    for (int x = 0; x < kQTiles; ++x) {
      mbar_init(s_full + 8 * x, 1);
      mbar_init(p_full + 8 * x, 4 * kSplit);
      mbar_init(o_full + 8 * x, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ================================ TMA producer ================================
    // The whole warp walks the chunk table (lane k: piece k of a tile, loaded ahead so the load
    // latency hides behind the barrier waits); lane 0 issues the TMAs.
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy));
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.kv)) : "memory");
      mbar_expect_tx(q_full, uint32_t(nq * LY::QT));
      for (int x = 0; x < nq; ++x)
        for (int h = 0; h < HALVES; ++h)  // box {64, group heads, 1 half, 128/group rows}
          tma_4d(sb + LY::off_q + x * LY::QT + h * kM * 128, &maps.q, 0, kvh * p.group, h, q_row0 + x * bp, q_full);
    }
    const int tp = p.T < kN ? p.T : kN;  // tokens per chunk piece
    const int32_t* trow = p.table + int64_t(req) * p.table_stride;
    auto pieces = [&](int t) { return (min(kN, last_key + 1 - t * kN) + tp - 1) / tp; };
    auto load_ent = [&](int t) {
      return (t < n_tiles && lane < pieces(t)) ? __ldg(trow + (t * kN + lane * tp) / p.T) : -1;
    };
    auto issue = [&](int t, int kv, int e) {
      const int ns = kv ? kVStages : kKStages;
      const int s = t % ns, round = t / ns;
      const uint32_t full = (kv ? v_full : k_full) + 8 * s, empty = (kv ? v_empty : k_empty) + 8 * s;
      const int npc = pieces(t);
      const uint32_t dst = sb + (kv ? LY::off_v : LY::off_k) + s * LY::TILE;
      // runs of consecutive chunk ids go as one box of 1/2/4/8 chunks (TMA issue cost is per box);
      // with rotated slabs a run also breaks at a rotation-group boundary (the slot changes there)
      const int prev = __shfl_up_sync(0xffffffffu, e, 1);
      unsigned starts = __ballot_sync(
          0xffffffffu, lane < npc && (lane == 0 || e != prev + 1 || p.T >= kN || !p.runs ||
                                      (p.rot && e % kRotGroup == 0)));
      if (lane == 0) {
        mbar_wait(empty, (round & 1) ^ 1);
        mbar_expect_tx(full, uint32_t(npc * tp * 128 * HALVES));
      }
      while (starts) {
        const int k = __ffs(starts) - 1;
        starts &= starts - 1;
        const int kend = starts ? __ffs(starts) - 1 : npc;
        const int c = __shfl_sync(0xffffffffu, e, k);
        if (lane == 0) {
          const int sl = slab_slot(c, p.layer, p.rot);
          if (p.T >= kN || !p.runs) {  // one box inside one chunk (128 tokens, or the chunk's T)
            for (int h = 0; h < HALVES; ++h)
              tma_5d(dst + h * kN * 128 + k * tp * 128, &maps.kv, 0, p.T >= kN ? (t * kN) % p.T : 0, h, kvh,
                     (c * p.L + sl) * 2 + kv, full, policy);
          } else {
            // run map dim 3: (kv, head) blocks over the whole pool; dim 4 steps one chunk
            const int c3 = (sl * 2 + kv) * p.Hkv + kvh;  // the run's slot: constant inside it
            for (int done = 0; done < kend - k;) {
              const int lg = min(3, 31 - __clz(kend - k - done));
              for (int h = 0; h < HALVES; ++h)
                tma_5d(dst + h * kN * 128 + (k + done) * tp * 128, &maps.run[lg], 0, 0, h, c3, c + done, full,
                       policy);
              done += 1 << lg;
            }
          }
        }
      }
      __syncwarp();
    };
    // order: K(0), K(1), V(0), K(2), V(1), ... — K one tile ahead of V
    int e_cur = load_ent(0), e_n1 = load_ent(1);
    issue(0, 0, e_cur);
    for (int t = 0; t < n_tiles; ++t) {
      const int e_after = load_ent(t + 2);  // in flight while this iteration waits
      if (t + 1 < n_tiles) issue(t + 1, 0, e_n1);
      issue(t, 1, e_cur);
      e_cur = e_n1;
      e_n1 = e_after;
    }
  } else if (warp == 1) {
    // ================================ MMA issuer (whole warp, one elected thread issues) =====
    {
      constexpr uint32_t id_s = idesc_bf16(kM, kN, false);
      constexpr uint32_t id_pv = idesc_bf16(kM, D, true);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int x, int t) {  // S_x(t) = Q_x K(t)^T into TMEM columns [128x, 128x + 128)
        const uint32_t kb = sb + LY::off_k + (t % kKStages) * LY::TILE;
        const uint32_t qb = sb + LY::off_q + x * LY::QT;
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * (kM * 128) + (k & 3) * 32;
          umma(tmem + x * 128, desc_sw128(qb + off, 16), desc_sw128(kb + off, 16), id_s, k > 0);
        }
        umma_commit(s_full + 8 * x);
      };
      auto issue_pv = [&](int x, int t) {  // O_x += P_x(t) V(t), P_x from TMEM (S_x's columns)
        mbar_wait(p_full + 8 * x, t & 1);
        if (lane == 0) pf_stamp(p, t, 4 + 2 * x);
        tc_fence_after();
        const uint32_t vb = sb + LY::off_v + (t % kVStages) * LY::TILE;
#pragma unroll
        for (int k = 0; k < kN / 16; ++k)
          umma_ts(tmem + 256 + x * 128, tmem + x * 128 + k * 8, desc_sw128(vb + k * 2048, kN * 128), id_pv,
                  (t > 0 || k > 0) ? 1u : 0u);
      };
      mbar_wait(k_full, 0);
      tc_fence_after();
      for (int x = 0; x < nq; ++x) issue_s(x, 0);
      umma_commit(k_empty);
      for (int t = 0; t < n_tiles; ++t) {
        const bool more = t + 1 < n_tiles;
        mbar_wait(v_full + 8 * (t % kVStages), (t / kVStages) & 1);
        if (more) mbar_wait(k_full + 8 * ((t + 1) % kKStages), ((t + 1) / kKStages) & 1);
        for (int x = 0; x < nq; ++x) {
          issue_pv(x, t);
          if (x == nq - 1) umma_commit(v_empty + 8 * (t % kVStages));
          if (more) {
            issue_s(x, t + 1);  // in order after P_x(t) was read: S_x may overwrite P_x
            if (lane == 0) pf_stamp(p, t, 5 + 2 * x);
            if (x == nq - 1) umma_commit(k_empty + 8 * ((t + 1) % kKStages));
          } else {
            umma_commit(o_full + 8 * x);
          }
        }
      }
    }
  } else {
    // ================================ softmax ================================
    // warps 2..9 -> Q tile 0, 10..17 -> Q tile 1. Thread = TMEM lane = MMA row; the two warps of a
    // (Q tile, lane quarter) pair split the tile's 128 keys into halves h = 0 / 1 and exchange
    // their row maxima through shared memory (named barrier per pair), so twice as many warps
    // keep the SFU (16 exp2 per SM-cycle: the per-tile budget at full tensor rate) busy.
    const int sw = warp - 2;
    const int x = sw / (4 * kSplit);
    const int h = (sw / 4) % kSplit;
    const int quarter = warp & 3;           // TMEM lanes [32*quarter, 32*quarter + 32) (warp % 4 rule)
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = tmem + (uint32_t(quarter * 32) << 16);
    constexpr int KH = kN / kSplit;         // keys of this warp's half
    const uint32_t s_col = x * 128 + h * KH, p_col = x * 128 + h * (KH / 2), o_col = 256 + x * 128 + h * (D / kSplit);
    const int g = p.group;
    const int pos_idx = x * bp + row / g;
    const bool valid = pos_idx < n_valid;
    const int prow = valid ? p0 + pos_idx : p0;  // causal limit of this row
    [[maybe_unused]] const uint32_t pair_bar = 1 + x * 4 + quarter;  // named barrier of the split warps
    float* red = reinterpret_cast<float*>(smem + LY::off_red);
    auto red_at = [&](int par, int hh) -> float& { return red[((par * kQTiles + x) * kSplit + hh) * kM + row]; };
    if (x < nq) {
      float m_run = -INFINITY, l_run = 0.f;
      for (int t = 0; t < n_tiles; ++t) {
        // S_x(t) complete implies P_x(t-1).V(t-1) complete (commit order): O_x and P_x are free
        mbar_wait(s_full + 8 * x, t & 1);
        if (h == 0 && quarter == 0 && lane == 0) pf_stamp(p, t, 2 * x);
        tc_fence_after();
        float xs[KH];
#pragma unroll
        for (int c = 0; c < KH / 32; ++c) tmem_ld32(lane_addr + s_col + c * 32, reinterpret_cast<uint32_t*>(xs + 32 * c));
        tmem_wait_ld();
        if (x == 0 && h == 0 && quarter == 0 && lane == 0) pf_stamp(p, t, 8);
        const int lim = prow - t * kN - h * KH;  // keys j <= lim of this half are visible
        if (!__all_sync(0xffffffffu, lim >= KH - 1)) {  // diagonal / last tiles only
#pragma unroll
          for (int j = 0; j < KH; ++j)
            if (j > lim) xs[j] = -INFINITY;
        }
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = xs[i];
#pragma unroll
        for (int j = 8; j < KH; ++j) mx[j & 7] = fmaxf(mx[j & 7], xs[j]);
        const float m_half =
            fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        // exchange with the other half (parity-buffered: the partner is at most one tile apart);
        // the barrier also orders both halves' S loads before either overwrites S with P
        if constexpr (kSplit > 1) {
          red_at(t & 1, h) = m_half;
          asm volatile("bar.sync %0, %1;" ::"r"(pair_bar), "n"(32 * kSplit) : "memory");
        }
        if (x == 0 && h == 0 && quarter == 0 && lane == 0) pf_stamp(p, t, 9);
        const float m_tile = (kSplit > 1 ? fmaxf(m_half, red_at(t & 1, h ^ 1)) : m_half) * p.scale_log2;
        // lazy rescale: the reference max moves only when the tile max exceeds it by more than
        // the headroom (both halves see the same m_tile, so they decide alike); each warp
        // rescales its half of O_x's columns (tcgen05.ld/st are .aligned: warp-uniform branch)
        const bool grow = m_tile > m_run + kRescaleHeadroom;
        if (t > 0 && __any_sync(0xffffffffu, grow)) {
          const float alpha = grow ? ex2(m_run - m_tile) : 1.f;
          l_run *= alpha;
#pragma unroll 1
          for (int c = 0; c < D / kSplit / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(lane_addr + o_col + c * 16, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st16(lane_addr + o_col + c * 16, o);
          }
        }
        if (grow) m_run = m_tile;
        float2 sm[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                        make_float2(0.f, 0.f)};
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m_run, -m_run);
        // exponentials, packed to bf16 pairs and stored as P_x's columns [32h, 32h + 32) (keys
        // 64h .. 64h + 63; the A operand of P.V, read from TMEM); scaling and sums on fp32 pairs
#pragma unroll
        for (int c = 0; c < KH / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float2 y = ffma2(make_float2(xs[32 * c + j], xs[32 * c + j + 1]), sc2, nm2);
            float a, b;
            if ((((32 * c + j) >> 1) & 7) < EMU) {  // this pair on the FMA pipe
              const float2 e = ex2_fma2(y);
              a = e.x;
              b = e.y;
            } else {
              a = ex2(y.x);
              b = ex2(y.y);
            }
            sm[(j >> 1) & 3] = fadd2(sm[(j >> 1) & 3], make_float2(a, b));
            pk[j / 2] = pack_bf16(a, b);
          }
          tmem_st16(lane_addr + p_col + c * 16, pk);
        }
        l_run += ((sm[0].x + sm[0].y) + (sm[1].x + sm[1].y)) + ((sm[2].x + sm[2].y) + (sm[3].x + sm[3].y));
        if (x == 0 && h == 0 && t == n_tiles - 1) {  // V rows past the last visible key may hold anything
          const int need = last_key + 1 - t * kN;
          // after the tile's TMA has landed: its last chunk piece may cover rows >= need, and S(t)
          // complete does not imply V(t) complete (V is loaded one tile behind K)
          mbar_wait(v_full + 8 * (t % kVStages), (t / kVStages) & 1);
          if (row >= need) {
            uint8_t* vrow = smem + LY::off_v + (t % kVStages) * LY::TILE + row * 128;
#pragma unroll
            for (int hf = 0; hf < HALVES; ++hf)
#pragma unroll
              for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(vrow + hf * kN * 128 + c * 16) = make_uint4(0, 0, 0, 0);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        tmem_wait_st();
        if (x == 0 && h == 0 && quarter == 0 && lane == 0) pf_stamp(p, t, 10);
        tc_fence_before();
        __syncwarp();
        if (h == 0 && quarter == 0 && lane == 0) pf_stamp(p, t, 2 * x + 1);
        if (lane == 0) mbar_arrive(p_full + 8 * x);
      }
      // ---- epilogue: O_x / (l_h0 + l_h1) -> bf16 -> out[q_row0 + pos][kvh*group + head][h half] ----
      float l_other = 0.f;
      if constexpr (kSplit > 1) {
        red_at(n_tiles & 1, h) = l_run;
        asm volatile("bar.sync %0, %1;" ::"r"(pair_bar), "n"(32 * kSplit) : "memory");
        l_other = red_at(n_tiles & 1, h ^ 1);
      }
      const float inv = 1.f / (l_run + l_other);
      mbar_wait(o_full + 8 * x, 0);
      tc_fence_after();
      __nv_bfloat16* dst = p.out + (int64_t(q_row0 + pos_idx) * p.Hq + kvh * g + row % g) * D + h * (D / kSplit);
#pragma unroll
      for (int c = 0; c < D / kSplit / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(lane_addr + o_col + c * 32, o);
        tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(o[e + 0]) * inv, __uint_as_float(o[e + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(o[e + 4]) * inv, __uint_as_float(o[e + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(o[e + 6]) * inv, __uint_as_float(o[e + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + c * 32 + e) = v;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

template <int D, int EMU>
cudaError_t launch_de(const PrefillMaps& maps, const PParams& prm, int n_work, cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};  // per device (function attributes are per context)
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(prefill_kernel<D, EMU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Layout<D>::bytes);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  prefill_kernel<D, EMU><<<n_work, kThreads, Layout<D>::bytes, s>>>(maps, prm);
  return cudaGetLastError();
}

constexpr int kDefaultEmu = 2;  // 2 of every 8 pairs on the FMA pipe: +2-4% over 0 (tools/pf_split_emu.sh)
template <int D>
cudaError_t launch_d(const PrefillMaps& maps, const PParams& prm, int n_work, cudaStream_t s) {
  const char* v = std::getenv("ELLM_PF_EMU");  // measurement knob: 0, 1, 2 or 3 pairs of every 8
  const int emu = v ? std::atoi(v) : kDefaultEmu;
  switch (emu) {
    case 0: return launch_de<D, 0>(maps, prm, n_work, s);
    case 1: return launch_de<D, 1>(maps, prm, n_work, s);
    case 3: return launch_de<D, 3>(maps, prm, n_work, s);
    default: return launch_de<D, 2>(maps, prm, n_work, s);
  }
}

}  // namespace

cudaError_t encode_prefill_kv_maps(PrefillMaps* m, void* pool_base, int64_t max_chunks, const AttnShape& sh,
                                   int64_t chunk_bytes) {
  const Driver& d = driver();
  if (!d.ok) return cudaErrorNotSupported;
  const int D = sh.D, halves = D / 64;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  {  // {64 d-elements, T tokens, d/64 halves, Hkv heads, chunk*L*2 + layer*2 + kv}; box 128 tokens
    cuuint64_t dims[5] = {64, cuuint64_t(sh.T), cuuint64_t(halves), cuuint64_t(sh.Hkv),
                          cuuint64_t(max_chunks) * sh.L * 2};
    cuuint64_t strides[4] = {cuuint64_t(D) * 2, 128, cuuint64_t(sh.T) * D * 2, cuuint64_t(sh.Hkv) * sh.T * D * 2};
    cuuint32_t box[5] = {64, cuuint32_t(sh.T < kN ? sh.T : kN), 1, 1, 1};
    if (d.tensorMapEncodeTiled(&m->kv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, pool_base, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  // runs of consecutive chunks (inside one rotation group when slabs are rotated):
  // {64, T, d/64, (slot*2 + kv)*Hkv + head, chunk}; box 1/2/4/8 chunks
  m->runs = 0;
  for (int lg = 0; lg < 4; ++lg) {
    cuuint64_t dims[5] = {64, cuuint64_t(sh.T), cuuint64_t(halves), cuuint64_t(sh.L) * 2 * sh.Hkv,
                          cuuint64_t(max_chunks)};
    cuuint64_t strides[4] = {cuuint64_t(D) * 2, 128, cuuint64_t(sh.T) * D * 2, cuuint64_t(chunk_bytes)};
    cuuint32_t box[5] = {64, cuuint32_t(sh.T < kN ? sh.T : kN), 1, 1, cuuint32_t(1) << lg};
    if (d.tensorMapEncodeTiled(&m->run[lg], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, pool_base, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaSuccess;  // no run maps: one box per chunk through m->kv (runs = 0)
  }
  m->runs = 1;
  return cudaSuccess;
}

cudaError_t encode_prefill_q_map(PrefillMaps* m, const AttnShape& sh, const void* q, int64_t q_rows) {
  const Driver& d = driver();
  if (!d.ok) return cudaErrorNotSupported;
  const int D = sh.D, halves = D / 64;
  // q: {64 d-elements, Hq heads, d/64 halves, rows}; box = (group heads) x (128/group rows)
  cuuint64_t dims[4] = {64, cuuint64_t(sh.Hq), cuuint64_t(halves), cuuint64_t(q_rows)};
  cuuint64_t strides[3] = {cuuint64_t(D) * 2, 128, cuuint64_t(sh.Hq) * D * 2};
  cuuint32_t box[4] = {64, cuuint32_t(sh.group), 1, cuuint32_t(kM / sh.group)};
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (d.tensorMapEncodeTiled(&m->q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(q), dims, strides, box,
                             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  return cudaSuccess;
}

cudaError_t launch_prefill_attention(const PrefillMaps& maps, const AttnShape& sh, const int32_t* work, int32_t n_work, const int32_t* table,
                                     int32_t table_stride, int32_t layer, void* out, float scale,
                                     cudaStream_t s, void* trace) {
  PParams prm;
  prm.work = reinterpret_cast<const int4*>(work);
  prm.table = table;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.table_stride = table_stride;
  prm.Hq = sh.Hq;
  prm.group = sh.group;
  prm.T = sh.T;
  prm.Hkv = sh.Hkv;
  prm.L = sh.L;
  prm.layer = layer;
  prm.rot = sh.rot;
  prm.runs = maps.runs;
  prm.scale_log2 = scale * 1.4426950408889634f;
  prm.trace = static_cast<unsigned long long*>(trace);
  if (n_work == 0) return cudaSuccess;
  return sh.D == 128 ? launch_d<128>(maps, prm, n_work, s) : launch_d<64>(maps, prm, n_work, s);
}

}  // namespace ellm

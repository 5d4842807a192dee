// hbm_read.cu — practical read-only HBM bandwidth on this B200 (roofline reference for the
// attention kernel, which only reads KV). Variants:
//   ldg   : grid-stride LDG.128, 8 independent loads in flight per thread
//   bulk  : persistent CTA per SM, one thread streams cp.async.bulk (1-D TMA) of STAGE bytes
//           into an NST-deep mbarrier ring; 8 warps release stages (no compute)
// Usage: hbm_read [GiB]   -> prints one JSON line per variant
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void ldg_kernel(const uint4* __restrict__ p, int64_t n, uint32_t* out) {
  uint32_t acc = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(p + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  for (; i < n; i += stride) { uint4 v = __ldcs(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// STRIDE > 0: unit u reads STAGE bytes at (u % per) * STRIDE + (u / per) * STAGE, i.e. 64 KiB
// slabs scattered at 2 MiB strides like the (chunk, layer) slabs of the pool.
template <int STAGE, int NST, int64_t STRIDE = 0>
__global__ void __launch_bounds__(288, 1) bulk_kernel(const uint8_t* __restrict__ p, int64_t bytes, uint32_t* out,
                                                      uint64_t* times = nullptr) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NST * STAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su32(bar + NST + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t units = bytes / STAGE;
  const int64_t u0 = int64_t(blockIdx.x) * units / gridDim.x, u1 = int64_t(blockIdx.x + 1) * units / gridDim.x;
  if (warp == 8) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int64_t u = u0; u < u1; ++u) {
        asm volatile("{.reg .pred q; W1: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W1;}" ::"r"(su32(bar + NST + s)), "r"(ph ^ 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + s)), "r"(STAGE));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sm + s * STAGE)),
                     "l"(p + (STRIDE ? (u % (bytes / STRIDE)) * STRIDE + (u / (bytes / STRIDE)) * STAGE : u * STAGE)),
                     "r"(STAGE), "r"(su32(bar + s)) : "memory");
        if (++s == NST) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  int s = 0; uint32_t ph = 0; uint32_t acc = 0;
  for (int64_t u = u0; u < u1; ++u) {
    asm volatile("{.reg .pred q; W2: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W2;}" ::"r"(su32(bar + s)), "r"(ph));
    acc ^= reinterpret_cast<const uint32_t*>(sm + s * STAGE)[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar + NST + s)));
    if (++s == NST) { s = 0; ph ^= 1; }
  }
  if (acc == 0x12345678u) out[0] = acc;
  if (times && threadIdx.x == 0) times[blockIdx.x] = gtimer();
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

template <int STAGE, int NST, int64_t STRIDE = 0>
void run_bulk(const uint8_t* d, int64_t bytes, uint32_t* o, int sms) {
  const int smem = NST * STAGE + 2 * 8 * NST;
  cudaFuncSetAttribute(bulk_kernel<STAGE, NST, STRIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint64_t* times;
  cudaMalloc(&times, sms * 8);
  float ms = time_it([&] { bulk_kernel<STAGE, NST, STRIDE><<<sms, 288, smem>>>(d, bytes, o, times); }, 5);
  // CTA finish-time spread of the last launch (globaltimer, ns)
  uint64_t h[1024];
  cudaMemcpy(h, times, sms * 8, cudaMemcpyDeviceToHost);
  uint64_t lo = h[0], hi = h[0];
  double mean = 0;
  for (int i = 0; i < sms; ++i) { lo = h[i] < lo ? h[i] : lo; hi = h[i] > hi ? h[i] : hi; mean += h[i]; }
  mean /= sms;
  printf("{\"variant\": \"bulk\", \"stage_kib\": %d, \"stages\": %d, \"stride\": %lld, \"gbs\": %.1f, "
         "\"finish_spread_us\": %.1f, \"mean_minus_first_us\": %.1f, \"kernel_us\": %.1f, \"err\": \"%s\"}\n",
         STAGE / 1024, NST, (long long)STRIDE, bytes / (ms * 1e-3) / 1e9, (hi - lo) / 1e3, (mean - lo) / 1e3, ms * 1e3,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(times);
}

int main(int argc, char** argv) {
  double gib = argc > 1 ? atof(argv[1]) : 8.0;
  int64_t bytes = int64_t(gib * (1 << 30));
  uint8_t* d; uint32_t* o;
  cudaMalloc(&d, bytes); cudaMalloc(&o, 64);
  cudaMemset(d, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mult : {4, 8, 16}) {
    float ms = time_it([&] { ldg_kernel<<<sms * mult, 256>>>((const uint4*)d, bytes / 16, o); }, 5);
    printf("{\"variant\": \"ldg\", \"blocks_per_sm\": %d, \"gbs\": %.1f}\n", mult, bytes / (ms * 1e-3) / 1e9);
  }
  run_bulk<65536, 3>(d, bytes, o, sms);
  run_bulk<32768, 6>(d, bytes, o, sms);
  run_bulk<16384, 12>(d, bytes, o, sms);
  run_bulk<32768, 4>(d, bytes, o, sms);
  run_bulk<65536, 2>(d, bytes, o, sms);
  run_bulk<65536, 3, 2 << 20>(d, bytes, o, sms);
  run_bulk<65536, 2, 2 << 20>(d, bytes, o, sms);
  run_bulk<32768, 6, 2 << 20>(d, bytes, o, sms);
  return 0;
}

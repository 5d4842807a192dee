// TMEM read / write throughput on this B200 (f4 design input): W warps (W/4 per TMEM lane
// quarter) each load 128 fp32 columns of their 32 lanes (tcgen05.ld.32x32b.x32 x4, then
// tcgen05.wait::ld) ITERS times; bytes per SM-cycle = W*32*128*4*ITERS / cycles. Same for
// tcgen05.st. nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include <cstdint>

#define R32(i) "=r"(r[i])
__device__ __forceinline__ void ld32(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : R32(0), R32(1), R32(2), R32(3), R32(4), R32(5), R32(6), R32(7), R32(8), R32(9), R32(10), R32(11),
                 R32(12), R32(13), R32(14), R32(15), R32(16), R32(17), R32(18), R32(19), R32(20), R32(21), R32(22),
                 R32(23), R32(24), R32(25), R32(26), R32(27), R32(28), R32(29), R32(30), R32(31)
               : "r"(a));
}
#define W32(i) "r"(r[i])
__device__ __forceinline__ void st32(uint32_t a, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
               W32(0), W32(1), W32(2), W32(3), W32(4), W32(5), W32(6), W32(7), W32(8), W32(9), W32(10), W32(11),
               W32(12), W32(13), W32(14), W32(15), W32(16), W32(17), W32(18), W32(19), W32(20), W32(21), W32(22),
               W32(23), W32(24), W32(25), W32(26), W32(27), W32(28), W32(29), W32(30), W32(31)
               : "memory");
}

template <bool STORE>
__global__ void tmem_kernel(int iters, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        uint32_t(__cvta_generic_to_shared(&slot))) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const uint32_t lane_addr = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 128 % 512);
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * i;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < 4; ++c) {
      if (STORE) st32(lane_addr + c * 32, r);
      else ld32(lane_addr + c * 32, r);
    }
    if (STORE) {
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += r[it & 31];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 8 * 148);
  cudaMalloc(&sink, 4 * 148 * 512);
  const int iters = 2000;
  for (int store = 0; store < 2; ++store)
    for (int warps : {4, 8, 16}) {
      if (store) tmem_kernel<true><<<148, warps * 32>>>(iters, cyc, sink);
      else tmem_kernel<false><<<148, warps * 32>>>(iters, cyc, sink);
      unsigned long long h[148];
      cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
      double bytes = double(warps) * 32 * 128 * 4 * iters;
      printf("%s warps=%2d: %.1f B/cycle/SM (%llu cycles)\n", store ? "tcgen05.st" : "tcgen05.ld", warps,
             bytes / double(h[0]), h[0]);
    }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}

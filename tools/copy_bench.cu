// copy_bench.cu — tuning the whole-chunk copy used by migrate (D2D) and swap (D2H / H2D):
// loads in flight per lane x blocks per SM, over 1024 scattered 2 MiB chunks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

template <int LOADS>
__global__ void __launch_bounds__(256) copy_kernel(uint8_t* __restrict__ dst_base, const int* __restrict__ dst_idx,
                                                   const uint8_t* __restrict__ src_base,
                                                   const int* __restrict__ src_idx, int n, long long chunk) {
  constexpr int UNIT = LOADS * 32 * 16;
  const int lane = threadIdx.x & 31;
  const long long upc = chunk / UNIT, total = (long long)n * upc;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total; w += warps) {
    const long long i = w / upc, off = (w % upc) * UNIT;
    const uint4* s = reinterpret_cast<const uint4*>(src_base + (long long)src_idx[i] * chunk + off);
    uint4* d = reinterpret_cast<uint4*>(dst_base + (long long)dst_idx[i] * chunk + off);
    uint4 v[LOADS];
#pragma unroll
    for (int k = 0; k < LOADS; ++k) v[k] = __ldcs(s + k * 32 + lane);
#pragma unroll
    for (int k = 0; k < LOADS; ++k) __stcs(d + k * 32 + lane, v[k]);
  }
}

template <int LOADS>
void run(const char* what, uint8_t* dst, const int* di, const uint8_t* src, const int* si, int n, long long chunk,
         int sms, int mult) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  copy_kernel<LOADS><<<sms * mult, 256>>>(dst, di, src, si, n, chunk);
  cudaDeviceSynchronize();
  float best = 1e9f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    copy_kernel<LOADS><<<sms * mult, 256>>>(dst, di, src, si, n, chunk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  const double bytes = (double)n * chunk;
  printf("{\"what\": \"%s\", \"loads\": %d, \"blocks_per_sm\": %d, \"gbs_moved\": %.1f, \"err\": \"%s\"}\n", what, LOADS,
         mult, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main() {
  const int n = 1024;
  const long long chunk = 2 << 20;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t *pool, *host, *hdev;
  cudaMalloc(&pool, 2 * n * chunk);
  cudaHostAlloc(&host, n * chunk, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&hdev, host, 0);
  std::vector<int> src(n), dst(n), slot(n);
  std::iota(src.begin(), src.end(), 0);
  std::iota(slot.begin(), slot.end(), 0);
  std::mt19937 g(1);
  std::shuffle(src.begin(), src.end(), g);
  for (int i = 0; i < n; ++i) dst[i] = n + i;
  int *dsrc, *ddst, *dslot;
  cudaMalloc(&dsrc, n * 4);
  cudaMalloc(&ddst, n * 4);
  cudaMalloc(&dslot, n * 4);
  cudaMemcpy(dsrc, src.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ddst, dst.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dslot, slot.data(), n * 4, cudaMemcpyHostToDevice);
  for (int mult : {1, 2, 4, 8}) {
    run<4>("d2d", pool, ddst, pool, dsrc, n, chunk, sms, mult);
    run<8>("d2d", pool, ddst, pool, dsrc, n, chunk, sms, mult);
    run<16>("d2d", pool, ddst, pool, dsrc, n, chunk, sms, mult);
  }
  for (int mult : {1, 2, 4}) {
    run<8>("d2h", hdev, dslot, pool, dsrc, n, chunk, sms, mult);
    run<16>("d2h", hdev, dslot, pool, dsrc, n, chunk, sms, mult);
    run<8>("h2d", pool, dsrc, hdev, dslot, n, chunk, sms, mult);
    run<16>("h2d", pool, dsrc, hdev, dslot, n, chunk, sms, mult);
  }
  return 0;
}

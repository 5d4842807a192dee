// slab_read.cu — read-only HBM microbenchmark with the pool's per-layer access pattern:
// for one layer l, read the slab [c*chunk + l*slab, +slab) of every chunk c (CTAs take
// contiguous ranges of chunks, 64 KiB bulk copies into a 3-stage mbarrier ring, like the
// attention kernel's producer). Isolates how the chunk stride (= L * slab) and the layer offset
// affect achieved bandwidth, with plain cudaMalloc memory (no VMM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/slab_read tools/slab_read.cu
//   tools/slab_read <pool GiB>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

static __device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

constexpr int STAGE = 65536, NST = 3;

__global__ void __launch_bounds__(288, 1) slab_kernel(const uint8_t* __restrict__ p, int64_t n_chunks, int64_t chunk,
                                                      int64_t slab, int64_t layer, int64_t rot, uint32_t* out) {
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
  const int64_t per = slab / STAGE;  // stages per slab
  const int64_t units = n_chunks * per;
  const int64_t u0 = int64_t(blockIdx.x) * units / gridDim.x, u1 = int64_t(blockIdx.x + 1) * units / gridDim.x;
  const int64_t L = chunk / slab;
  if (warp == 8) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int64_t u = u0; u < u1; ++u) {
        const int64_t c = u / per, k = u % per;
        const int64_t lpos = rot ? (layer + c / rot) % L : layer;  // rot = G: slot rotated per group of G chunks
        const uint8_t* src = p + c * chunk + lpos * slab + k * STAGE;
        asm volatile("{.reg .pred q; W1: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W1;}" ::"r"(su32(bar + NST + s)), "r"(ph ^ 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + s)), "r"(STAGE));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sm + s * STAGE)), "l"(src), "r"(STAGE), "r"(su32(bar + s)) : "memory");
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
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 150.0;
  const int64_t bytes = int64_t(gib * double(1ll << 30));
  uint8_t* d; uint32_t* o;
  if (cudaMalloc(&d, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&o, 64);
  cudaMemset(d, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = NST * STAGE + 2 * 8 * NST;
  cudaFuncSetAttribute(slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int64_t slab : {int64_t(65536), int64_t(131072)}) {
    for (int L : (argc > 2 ? std::vector<int>{32, 40, 80} : std::vector<int>{32, 36, 40, 48, 56, 64, 72, 80})) {
      const int64_t chunk = slab * L;
      const int64_t n = bytes / chunk;
      for (int rot : {0, 8, 16, 32, 64}) {
        double best = 0, worst = 1e30;
        for (int layer : {0, 5, 17, L - 1}) {
          float bms = 1e30f;
          for (int r = 0; r < 4; ++r) {
            cudaEventRecord(a);
            slab_kernel<<<sms, 288, smem>>>(d, n, chunk, slab, layer, rot, o);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < bms) bms = ms;
          }
          const double gbs = double(n * slab) / (bms * 1e-3) / 1e9;
          best = gbs > best ? gbs : best; worst = gbs < worst ? gbs : worst;
        }
        printf("{\"slab_kib\": %lld, \"L\": %d, \"chunk_mib\": %.2f, \"rot_group\": %d, \"n_chunks\": %lld, \"gbs_worst_layer\": %.0f, \"gbs_best_layer\": %.0f, \"err\": \"%s\"}\n",
               (long long)(slab >> 10), L, chunk / 1048576.0, rot, (long long)n, worst, best, cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
      }
    }
  }
  return 0;
}

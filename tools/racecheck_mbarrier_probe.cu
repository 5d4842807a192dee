// Is racecheck's report on paged_attn_kernel's stage metadata (written by the producer warp
// after mbarrier-waiting on `empty`, read by consumer warps after mbarrier-waiting on `full`) a
// property of the mbarrier hand-off itself? This kernel is that hand-off and nothing else: one
// producer warp writes meta[stage] then arrives on full[stage]; 8 consumer warps wait full[stage],
// read meta[stage], arrive on empty[stage]; the producer waits empty[stage] before rewriting it.
// A correct ring by construction (the checksum is verified). Run under
//   compute-sanitizer --tool racecheck ./racecheck_mbarrier_probe
// nvcc -gencode arch=compute_100a,code=sm_100a -o racecheck_mbarrier_probe racecheck_mbarrier_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
               ::"r"(bar), "r"(par) : "memory");
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

constexpr int NST = 3, ITERS = 64, CONS = 8;
__global__ void ring(unsigned long long* out) {
  __shared__ int meta[NST];
  __shared__ alignas(8) uint64_t full[NST], empty[NST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(CONS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CONS) {
    if (lane == 0)
      for (int i = 0; i < ITERS; ++i) {
        const int s = i % NST;
        wait(sa(&empty[s]), ((i / NST) & 1) ^ 1);
        meta[s] = i;
        arrive(sa(&full[s]));
      }
    return;
  }
  unsigned long long sum = 0;
  for (int i = 0; i < ITERS; ++i) {
    const int s = i % NST;
    wait(sa(&full[s]), (i / NST) & 1);
    sum += meta[s];
    __syncwarp();
    if (lane == 0) arrive(sa(&empty[s]));
  }
  if (lane == 0) atomicAdd(out, sum);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  ring<<<4, (CONS + 1) * 32>>>(d);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const unsigned long long want = 4ull * CONS * (ITERS * (ITERS - 1) / 2);
  printf("checksum %llu (want %llu) %s\n", h, want, h == want ? "ok" : "MISMATCH");
  return h == want ? 0 : 1;
}

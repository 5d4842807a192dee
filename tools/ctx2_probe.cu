// Does C3's swap interference depend on the CUDA context that issues the host->device copy?
// (DESIGN §5 C3, §10.) A streaming read kernel with the decode attention's access pattern — one
// 64 KiB slab of every 2 MiB page of a VMM-mapped footprint per launch, the slab offset moving
// with the "layer" — is timed with CUDA events alone and while pinned host -> device copies run
//   same:      on a second stream of the same (primary) context,
//   ctx2:      on a stream of a second context on the same device (cuCtxCreate), driven by its
//              own thread,
//   ctx2pool:  the same, copying into the read footprint itself (VMM memory mapped in the process
//              and granted to the device, so it is addressable from the second context too).
// Prints one line per variant: mean launch µs, slowdown, achieved read GB/s, copy GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ctx2_probe tools/ctx2_probe.cu -lcuda
//   tools/ctx2_probe [footprint_GiB=128] [launches=64]
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#define CK(x)                                                                                   \
  do {                                                                                          \
    CUresult r_ = (x);                                                                          \
    if (r_ != CUDA_SUCCESS) {                                                                   \
      const char* s_;                                                                           \
      cuGetErrorString(r_, &s_);                                                                \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, s_);                            \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

constexpr size_t kPage = 2u << 20, kSlab = 64u << 10;

// one CTA-wide 16 B-vector sweep over slab `layer` of pages [b*per, (b+1)*per)
__global__ void slab_read(const uint4* base, size_t pages, int layer, unsigned long long* sink) {
  const size_t per = (pages + gridDim.x - 1) / gridDim.x;
  const size_t p0 = blockIdx.x * per, p1 = p0 + per < pages ? p0 + per : pages;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t pg = p0; pg < p1; ++pg) {
    const uint4* s = base + (pg * kPage + size_t(layer) * kSlab) / 16;
#pragma unroll 4
    for (int i = threadIdx.x; i < int(kSlab / 16); i += blockDim.x) {
      uint4 v;
      asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s + i));
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x9e3779b9u) atomicAdd(sink, 1ull);
}

int main(int argc, char** argv) {
  const size_t gib = argc > 1 ? atol(argv[1]) : 128;
  const int launches = argc > 2 ? atoi(argv[2]) : 64;
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext prim;
  CK(cuDevicePrimaryCtxRetain(&prim, dev));
  CK(cuCtxSetCurrent(prim));
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);

  // footprint: VMM, 2 GiB handles, one VA range, access granted to the device
  const size_t bytes = gib << 30, unit = 2ull << 30;
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, bytes, 0, 0, 0));
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  for (size_t off = 0; off < bytes; off += unit) {
    CUmemGenericAllocationHandle h;
    CK(cuMemCreate(&h, unit, &prop, 0));
    CK(cuMemMap(va + off, unit, 0, h, 0));
    CK(cuMemRelease(h));
  }
  CUmemAccessDesc ad = {};
  ad.location = prop.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(va, bytes, &ad, 1));
  CK(cuMemsetD8(va, 1, bytes));
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const size_t pages = bytes / kPage;

  // host side: 1 GiB pinned (portable: usable from every context)
  const size_t cbytes = 1ull << 30;
  void* host;
  CK(cuMemHostAlloc(&host, cbytes, CU_MEMHOSTALLOC_PORTABLE));
  CUdeviceptr dsame;
  CK(cuMemAlloc(&dsame, cbytes));
  CK(cuCtxSynchronize());

  CUcontext ctx2;
#if CUDA_VERSION >= 12050
  CK(cuCtxCreate_v4(&ctx2, nullptr, 0, dev));
#else
  CK(cuCtxCreate(&ctx2, 0, dev));
#endif
  CUdeviceptr d2;
  CK(cuMemAlloc(&d2, cbytes));
  CUstream s2;
  CK(cuStreamCreate(&s2, CU_STREAM_NON_BLOCKING));
  CK(cuCtxSetCurrent(prim));
  CUstream sside;
  CK(cuStreamCreate(&sside, CU_STREAM_NON_BLOCKING));
  cudaStream_t sk;
  cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);

  auto run = [&](const char* name, int mode) {
    std::atomic<bool> stop{false};
    std::atomic<long> copied{0};
    std::thread th;
    if (mode > 0) {
      th = std::thread([&] {
        CUcontext c = mode == 1 ? prim : ctx2;
        CUstream s = mode == 1 ? sside : s2;
        CUdeviceptr dst = mode == 1 ? dsame : mode == 2 ? d2 : va + bytes / 3;
        CK(cuCtxSetCurrent(c));
        while (!stop.load()) {
          for (int i = 0; i < 2; ++i) CK(cuMemcpyHtoDAsync(dst, host, cbytes, s));
          CK(cuStreamSynchronize(s));
          copied += 2;
        }
      });
      std::this_thread::sleep_for(std::chrono::milliseconds(200));
    }
    CK(cuCtxSetCurrent(prim));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const long c0 = copied.load();
    auto t0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0, sk);
    for (int l = 0; l < launches; ++l)
      slab_read<<<nsm * 4, 512, 0, sk>>>(reinterpret_cast<const uint4*>(va), pages, l % 32, sink);
    cudaEventRecord(e1, sk);
    cudaEventSynchronize(e1);
    auto t1 = std::chrono::steady_clock::now();
    const long c1 = copied.load();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    stop = true;
    if (th.joinable()) th.join();
    const double wall = std::chrono::duration<double>(t1 - t0).count();
    const double us = ms * 1e3 / launches;
    printf("%-9s footprint %3zu GiB: %8.1f us/launch  read %6.0f GB/s  copy ~%5.1f GB/s\n", name, gib, us,
           double(pages) * kSlab / (us * 1e-6) / 1e9, double(c1 - c0) * cbytes / wall / 1e9);
    fflush(stdout);
    return us;
  };
  run("warmup", 0);
  const double base = run("alone", 0);
  for (int rep = 0; rep < 2; ++rep) {
    printf("  same / alone %.3f\n", run("same", 1) / base);
    printf("  ctx2 / alone %.3f\n", run("ctx2", 2) / base);
    printf("  ctx2pool / alone %.3f\n", run("ctx2pool", 3) / base);
    run("alone", 0);
  }
  return 0;
}

// vmm_bench.cu — latency of the CUDA VMM calls behind the pool (cuMemCreate / cuMemMap /
// cuMemSetAccess / cuMemUnmap / cuMemRelease) as a function of how they are batched and of
// the size of the reserved VA range. Prints one JSON line per variant.
#include <cuda.h>
#include <cuda_runtime.h>
#include <time.h>

#include <cstdio>
#include <vector>

static double now() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { printf("{\"err\": \"%s -> %d\"}\n", #x, int(r)); return; } } while (0)

static CUmemAllocationProp prop() {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = 0;
  return p;
}

// n handles of `bytes` each, mapped back to back into a reservation of `reserve` bytes.
static void run(const char* name, size_t bytes, int n, size_t reserve, bool access_once) {
  CUmemAllocationProp p = prop();
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, reserve, 0, 0, 0));
  std::vector<CUmemGenericAllocationHandle> h(n);
  double t0 = now();
  for (int i = 0; i < n; ++i) CK(cuMemCreate(&h[i], bytes, &p, 0));
  double t1 = now();
  for (int i = 0; i < n; ++i) CK(cuMemMap(va + size_t(i) * bytes, bytes, 0, h[i], 0));
  double t2 = now();
  if (access_once) {
    CK(cuMemSetAccess(va, size_t(n) * bytes, &acc, 1));
  } else {
    for (int i = 0; i < n; ++i) CK(cuMemSetAccess(va + size_t(i) * bytes, bytes, &acc, 1));
  }
  double t3 = now();
  for (int i = 0; i < n; ++i) CK(cuMemUnmap(va + size_t(i) * bytes, bytes));
  double t4 = now();
  for (int i = 0; i < n; ++i) CK(cuMemRelease(h[i]));
  double t5 = now();
  CK(cuMemAddressFree(va, reserve));
  printf("{\"variant\": \"%s\", \"handle_mib\": %zu, \"n\": %d, \"reserve_gib\": %.1f, \"create_us\": %.1f, "
         "\"map_us\": %.1f, \"setaccess_us_per_handle\": %.1f, \"unmap_us\": %.1f, \"release_us\": %.1f}\n",
         name, bytes >> 20, n, reserve / 1073741824.0, (t1 - t0) / n * 1e6, (t2 - t1) / n * 1e6,
         (t3 - t2) / n * 1e6, (t4 - t3) / n * 1e6, (t5 - t4) / n * 1e6);
  fflush(stdout);
}

int main() {
  cudaFree(0);
  const size_t MB2 = 2 << 20;
  run("per-chunk access, small VA", MB2, 1024, 1024 * MB2, false);
  run("one access, small VA", MB2, 1024, 1024 * MB2, true);
  run("per-chunk access, 130 GiB VA", MB2, 1024, size_t(130) << 30, false);
  run("one access, 130 GiB VA", MB2, 1024, size_t(130) << 30, true);
  run("64 MiB handles, one access", 64 * MB2 / 2, 32, 1024 * MB2, true);
  run("per-chunk access, 8192 chunks", MB2, 8192, 8192 * MB2, false);
  run("one access, 8192 chunks", MB2, 8192, 8192 * MB2, true);
  run("one access, 32768 chunks", MB2, 32768, 32768 * MB2, true);
  return 0;
}

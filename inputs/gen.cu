// gen.cu — CUDA twin of inputs/gen.py (the seeded counter-based input generator).
// Holds none of the method's arithmetic; shared by nothing in the product library.
// Built as inputs/libellm_inputs.so; bit-identity with gen.py is tested on the GPU.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return splitmix64(seed ^ (stream * 0xD1B54A32D192ED03ull));
}
__device__ __forceinline__ uint16_t bf16_from_hash(uint64_t h) {
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += int64_t((h >> (16 * i)) & 0xFFFF);
  float f = __fmul_rn(float(int32_t(s - 131070)), 3.0517578125e-05f);  // exact: * 2^-15
  uint32_t u = __float_as_uint(f);
  u = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
  return uint16_t(u);
}
__device__ __forceinline__ uint64_t kv_index(uint64_t r, uint64_t p, uint64_t l, uint64_t h, uint64_t e) {
  return (((((r << 21) | p) << 8 | l) << 8 | h) << 10) | e;
}
__device__ __forceinline__ uint64_t q_index(uint64_t r, uint64_t l, uint64_t h, uint64_t e) {
  return (((r << 8 | l) << 8 | h) << 10) | e;
}

// out[(row * nh + hi) * d + e] for rows = positions p0 .. p0+n-1 of request r, heads h0+hi.
__global__ void gen_kv_kernel(uint64_t seed, int32_t r, int64_t p0, int32_t n, int32_t l, int32_t kv,
                              int32_t h0, int32_t nh, int32_t d, int32_t group, int64_t needle_range,
                              uint16_t* out) {
  const uint64_t kkey = stream_key(seed, kv == 0 ? 1 : 2);
  const uint64_t qkey = stream_key(seed, 3);
  const uint64_t npkey = stream_key(seed, 4);
  const uint64_t nskey = stream_key(seed, 5);
  const int64_t total = int64_t(n) * nh * d;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t e = int32_t(i % d);
    const int32_t hi = int32_t((i / d) % nh);
    const int64_t row = i / (int64_t(d) * nh);
    const uint64_t p = uint64_t(p0 + row);
    const uint64_t h = uint64_t(h0 + hi);
    const uint64_t idx = kv_index(uint64_t(r), p, uint64_t(l), h, uint64_t(e));
    uint16_t v = bf16_from_hash(splitmix64(kkey + idx));
    if (needle_range > 0) {
      bool hit = false;
      for (int k = 0; k < 3; ++k) {
        uint64_t nidx = (((uint64_t(r) << 8 | uint64_t(l)) << 8 | h) << 2) | uint64_t(k);
        if (splitmix64(npkey + nidx) % uint64_t(needle_range) == p) hit = true;
      }
      if (hit) {
        if (kv == 0) {
          uint16_t q0 = bf16_from_hash(splitmix64(qkey + q_index(uint64_t(r), uint64_t(l), h * uint64_t(group), uint64_t(e))));
          v = (q0 & 0x7FFF) == 0 ? q0 : uint16_t(q0 + 0x0100);
        } else {
          v = (splitmix64(nskey + idx) & 1) ? 0xC040 : 0x4040;
        }
      }
    }
    out[i] = v;
  }
}

__global__ void gen_q_kernel(uint64_t seed, int32_t r, int32_t l, int32_t h0, int32_t nh, int32_t d, uint16_t* out) {
  const uint64_t qkey = stream_key(seed, 3);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < int64_t(nh) * d; i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t e = int32_t(i % d), hi = int32_t(i / d);
    out[i] = bf16_from_hash(splitmix64(qkey + q_index(uint64_t(r), uint64_t(l), uint64_t(h0 + hi), uint64_t(e))));
  }
}

int grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  return int(b < 4096 ? (b > 0 ? b : 1) : 4096);
}

}  // namespace

extern "C" {

// K (kv=0) / V (kv=1) rows of request r, positions [p0, p0+n), global kv-heads [h0, h0+nh).
int ellm_gen_kv(uint64_t seed, int32_t r, int64_t p0, int32_t n, int32_t l, int32_t kv, int32_t h0,
                int32_t nh, int32_t d, int32_t group, int64_t needle_range, void* out, void* stream) {
  int64_t total = int64_t(n) * nh * d;
  if (total <= 0) return 0;
  gen_kv_kernel<<<grid_for(total), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      seed, r, p0, n, l, kv, h0, nh, d, group, needle_range, static_cast<uint16_t*>(out));
  return cudaGetLastError() == cudaSuccess ? 0 : -9;
}

// Q of request r, layer l, global q-heads [h0, h0+nh) -> [nh, d].
int ellm_gen_q(uint64_t seed, int32_t r, int32_t l, int32_t h0, int32_t nh, int32_t d, void* out, void* stream) {
  gen_q_kernel<<<grid_for(int64_t(nh) * d), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      seed, r, l, h0, nh, d, static_cast<uint16_t*>(out));
  return cudaGetLastError() == cudaSuccess ? 0 : -9;
}

}

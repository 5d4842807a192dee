// Issue rate of MUFU.EX2 (ex2.approx.ftz.f32) and of the other softmax instructions per SM on
// this B200: W warps per SM each run ITERS x 32 independent operations; prints warp-instructions
// per SM-cycle. nvcc -gencode arch=compute_100a,code=sm_100a -o tools/mufu_bw tools/mufu_bw.cu
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void k(int iters, float* out, unsigned long long* cyc) {
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = -float(threadIdx.x + i) * 1e-3f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f00000001;" : "+f"(v[i]));
      if (OP == 2) {
        uint64_t x = *reinterpret_cast<uint64_t*>(&v[i & ~1]);
        if ((i & 1) == 0) {
          asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(x) : "l"(0x3F7FFFFF3F7FFFFFull));
          *reinterpret_cast<uint64_t*>(&v[i]) = x;
        }
      }
      if (OP == 3) {
        uint32_t r;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(__float_as_uint(v[i])));
        v[i] = __uint_as_float(r);
      }
      if (OP == 4) {  // F2FP: two fp32 -> packed bf16x2 (round to nearest even)
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[(i + 1) & 31]));
        v[i] = __uint_as_float(r ^ 0x3f803f80u);
      }
      if (OP == 5) {  // MUFU.EX2 and F2FP interleaved 1:1
        uint32_t r;
        if (i & 1) {
          asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[i - 1]));
          v[i] = __uint_as_float(r ^ 0x3f803f80u);
        } else {
          asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
        }
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 32; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 4 * 148 * 1024);
  cudaMalloc(&cyc, 8 * 148);
  const char* names[] = {"MUFU.EX2 f32", "FFMA", "FFMA2 (f32x2)", "MUFU.EX2 bf16x2", "F2FP bf16x2", "EX2+F2FP 1:1"};
  const int iters = 4096;
  for (int op = 0; op < 6; ++op)
    for (int warps : {4, 8, 16}) {
      switch (op) {
        case 0: k<0><<<148, warps * 32>>>(iters, out, cyc); break;
        case 1: k<1><<<148, warps * 32>>>(iters, out, cyc); break;
        case 2: k<2><<<148, warps * 32>>>(iters, out, cyc); break;
        case 3: k<3><<<148, warps * 32>>>(iters, out, cyc); break;
        case 4: k<4><<<148, warps * 32>>>(iters, out, cyc); break;
        case 5: k<5><<<148, warps * 32>>>(iters, out, cyc); break;
      }
      unsigned long long h[148];
      cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
      const double instr = double(warps) * iters * (op == 2 ? 16 : 32);
      printf("%-18s warps=%2d: %.2f warp-instr per SM-cycle\n", names[op], warps, instr / double(h[0]));
    }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

// FFMA issue-rate microbench on one SM: 3-register form vs immediate form vs FFMA2.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, float a, float b, int iters, long long* cyc) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 0.001f + i;
  float bb[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) bb[i] = b + i * 1e-3f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) acc[i] = fmaf(a, bb[i], acc[i]);                  // 3 registers
      else if (MODE == 1) acc[i] = fmaf(1.0001f, bb[i], acc[i]);       // immediate
    }
    if (MODE == 2) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        unsigned long long x, y, z;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(acc[i]), "f"(acc[i + 1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(bb[i]), "f"(bb[i + 1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(z) : "f"(a), "f"(a));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(x) : "l"(z), "l"(y));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(x));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMallocManaged(&out, 1 << 20); cudaMallocManaged(&cyc, 8);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    for (int mode = 0; mode < 3; ++mode) {
      if (mode == 0) k<0><<<1, 32 * warps>>>(out, 1.0001f, 0.5f, iters, cyc);
      if (mode == 1) k<1><<<1, 32 * warps>>>(out, 1.0001f, 0.5f, iters, cyc);
      if (mode == 2) k<2><<<1, 32 * warps>>>(out, 1.0001f, 0.5f, iters, cyc);
      cudaDeviceSynchronize();
      const double fmas = (double)iters * 16 * 32 * warps;
      printf("warps %2d mode %s: %.1f FMA/clk/SM\n", warps, mode == 0 ? "FFMA 3-reg" : mode == 1 ? "FFMA imm  " : "FFMA2     ",
             fmas / *cyc);
    }
  }
}

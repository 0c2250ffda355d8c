// Minimal tcgen05 kind::tf32 probe: D[128x64] = A[128x32] * B[64x32]^T with
// A, B in K-major SW128 shared-memory tiles, one CTA. Checks descriptor /
// commit / TMEM-load plumbing in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/tc_probe.cu -o tc_probe && ./tc_probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned int u32;
#define DEVI __device__ __forceinline__

DEVI u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
DEVI void mbar_init(u64* b, u32 n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(b)), "r"(n) : "memory"); }
DEVI bool mbar_try(u64* b, u32 parity) {
  u32 ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(smem_addr(b)), "r"(parity) : "memory");
  return ok != 0;
}
DEVI u64 sdesc(u32 saddr, int mode) {
  u64 d = (u64)((saddr & 0x3FFFFu) >> 4) | ((u64)1 << 16) | ((u64)(512 >> 4) << 32) | ((u64)4 << 61);
  if (mode & 1) d |= (u64)1 << 46;  // version
  return d;
}

__global__ void probe(const float* A, const float* B, float* D, int mode, int* status, int mma_warp, int col) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((unsigned long long)smem_raw + 1023) & ~1023ull);
  unsigned char* sa = sm;          // 128 x 32 fp32 = 16 KB
  unsigned char* sb = sm + 16384;  // 64 x 32 fp32 = 8 KB
  u64* bar = (u64*)(sm + 16384 + 8192);
  u64* bar2 = bar + 1;
  u32* tslot = (u32*)(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, c = e % 32, h = c >> 4, cl = c & 15;  // two 16-channel SW64 tiles
    *(float*)(sa + h * 8192 + (m >> 3) * 512 + (m & 7) * 64 + (((cl >> 2) ^ ((m >> 1) & 3)) << 4) + (cl & 3) * 4) = A[e];
  }
  for (int e = tid; e < 64 * 32; e += blockDim.x) {
    const int n = e / 32, c = e % 32, h = c >> 4, cl = c & 15;
    *(float*)(sb + h * 4096 + (n >> 3) * 512 + (n & 7) * 64 + (((cl >> 2) ^ ((n >> 1) & 3)) << 4) + (cl & 3) * 4) = B[e];
  }
  if (tid == 0) { mbar_init(bar, 1); mbar_init(bar2, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == mma_warp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_addr(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = *tslot;
  if (warp == mma_warp && (tid & 31) == 0) {
    const u32 idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(64 >> 3) << 17) | ((u32)(128 >> 4) << 24);
    for (int ks = 0; ks < 4; ++ks) {
      const u64 a = sdesc(smem_addr(sa) + (ks >> 1) * 8192 + (ks & 1) * 32, mode), b = sdesc(smem_addr(sb) + (ks >> 1) * 4096 + (ks & 1) * 32, mode);
      const u32 acc = ks > 0;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                   :: "r"(tmem + col), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_addr(bar)) : "memory");
    if (mode & 2) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_addr(bar2)) : "memory");
  }
  __syncwarp();
  // wait (bounded)
  long long t0 = clock64();
  bool ok = false;
  while (clock64() - t0 < 2000000000ll) { if (mbar_try(bar, 0)) { ok = true; break; } }
  if (!ok) { if (tid == 0) *status = 1; }
  if (ok && (mode & 2)) {
    ok = false; t0 = clock64();
    while (clock64() - t0 < 2000000000ll) { if (mbar_try(bar2, 0)) { ok = true; break; } }
    if (!ok && tid == 0) *status = 2;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (ok && warp < 4) {
    for (int c0 = 0; c0 < 64; c0 += 8) {
      u32 r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem + ((u32)(32 * warp) << 16) + col + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 8; ++i) D[(32 * warp + (tid & 31)) * 64 + c0 + i] = __uint_as_float(r[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == mma_warp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

int main(int argc, char** argv) {
  const int threads = argc > 1 ? atoi(argv[1]) : 128, mma_warp = argc > 2 ? atoi(argv[2]) : 0, col = argc > 3 ? atoi(argv[3]) : 0;
  printf("threads %d mma_warp %d col %d\n", threads, mma_warp, col);
  float *A, *B, *D; int* st;
  cudaMallocManaged(&A, 128 * 32 * 4); cudaMallocManaged(&B, 64 * 32 * 4); cudaMallocManaged(&D, 128 * 64 * 4);
  cudaMallocManaged(&st, 4);
  for (int i = 0; i < 128 * 32; ++i) A[i] = (float)((i * 7 + i / 32) % 13 - 6) / 8.f;
  for (int i = 0; i < 64 * 32; ++i) B[i] = (float)((i * 5) % 11 - 5) / 4.f;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int mode = 3; mode >= 0; --mode) {
    *st = 0;
    for (int i = 0; i < 128 * 64; ++i) D[i] = -999.f;
    probe<<<1, threads, 40000>>>(A, B, D, mode, st, mma_warp, col);
    cudaError_t e = cudaDeviceSynchronize();
    double err = 0; int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        double ref = 0;
        for (int k = 0; k < 32; ++k) ref += (double)A[m * 32 + k] * B[n * 32 + k];
        const double d = fabs(ref - D[m * 64 + n]);
        err = fmax(err, d);
        if (d > 1e-3 && bad++ < 3) printf("  m=%d n=%d got %f want %f\n", m, n, D[m * 64 + n], ref);
      }
    printf("mode %d (version bit %d): cuda=%s timeout=%d max_abs_err=%g\n", mode, mode & 1, cudaGetErrorString(e), *st, err);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}

// Probe: tcgen05 kind::tf32, M=64, N=64, both operands MN-major SW64 in
// shared memory, K = 128 (16 steps of 8 rows); D = A^T B read back with the
// M=64 TMEM layout (lanes 0-63: n < 32, lanes 64-127: n >= 32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/tc_probe_mn.cu -o tools/tc_probe_mn
#include <cmath>
#include <cstdio>
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
DEVI u64 desc(u32 saddr, u32 lbo, u32 sbo) {
  return (u64)((saddr & 0x3FFFFu) >> 4) | ((u64)(lbo >> 4) << 16) | ((u64)(sbo >> 4) << 32) | ((u64)1 << 46) | ((u64)4 << 61);
}
DEVI u32 sw64(int m, int chunk) { return (u32)((m >> 3) * 512 + (m & 7) * 64 + ((chunk ^ ((m >> 1) & 3)) << 4)); }

// A[k][m] (k = 0..127 rows, m = 0..63), B[k][n]; tile: block (col / 16) at 8 KB, row k at sw64.
__global__ void probe(const float* A, const float* B, float* D, int variant) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((unsigned long long)smem_raw + 1023) & ~1023ull);
  unsigned char* sa = sm;
  unsigned char* sb = sm + 32768;
  u64* bar = (u64*)(sm + 65536);
  u32* tslot = (u32*)(bar + 1);
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    const int k = e / 64, c = e % 64;
    u32 off;
    if (variant < 2) off = (c >> 4) * 8192 + sw64(k, (c & 15) >> 2) + (c & 3) * 4;      // MN-major
    else off = (k >> 4) * 4096 + sw64(c, (k & 15) >> 2) + (k & 3) * 4;                 // K-major [c][k]
    *(float*)(sa + off) = A[e];
    *(float*)(sb + off) = B[e];
  }
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"(smem_addr(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = *tslot;
  if (threadIdx.x == 0) {
    const u32 mn = variant < 2 ? 3u : 0u;
    const u32 idesc = (1u << 4) | (2u << 7) | (2u << 10) | (mn << 15) | ((u32)(64 >> 3) << 17) | ((u32)(64 >> 4) << 24);
    const u32 lbo = variant == 1 ? 512 : variant == 0 ? 8192 : 16, sbo = variant == 1 ? 8192 : 512;
    for (int s = 0; s < 16; ++s) {
      const u32 o = variant < 2 ? s * 512 : (s >> 1) * 4096 + (s & 1) * 32;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                   :: "r"(tmem), "l"(desc(smem_addr(sa) + o, lbo, sbo)), "l"(desc(smem_addr(sb) + o, lbo, sbo)),
                      "r"(idesc), "r"(s ? 1u : 0u) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_addr(bar)) : "memory");
  }
  __syncwarp();
  while (!mbar_try(bar, 0)) { }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 128) {
    const int w = threadIdx.x >> 5;
    for (int c0 = 0; c0 < 64; c0 += 8) {
      u32 r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem + ((u32)(32 * w) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 8; ++i) D[threadIdx.x * 64 + c0 + i] = __uint_as_float(r[i]);  // raw [lane][col]
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(tmem));
}

int main() {
  float *A, *B, *D;
  cudaMallocManaged(&A, 128 * 64 * 4); cudaMallocManaged(&B, 128 * 64 * 4); cudaMallocManaged(&D, 128 * 64 * 4);
  for (int i = 0; i < 128 * 64; ++i) { A[i] = (float)((i * 7 + i / 64) % 13 - 6) / 8.f; B[i] = (float)((i * 5 + 3) % 11 - 5) / 4.f; }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  for (int variant = 0; variant < 3; ++variant) {
    for (int i = 0; i < 128 * 64; ++i) D[i] = -999.f;
    probe<<<1, 128, 80000>>>(A, B, D, variant);
    cudaError_t e = cudaDeviceSynchronize();
    // want[m][n] = sum_k A[k][m] B[k][n]; assumed layout: lane = m + 64 (n >= 32), col = n % 32
    double err = 0; int shown = 0;
    for (int m = 0; m < 64; ++m)
      for (int n = 0; n < 64; ++n) {
        double want = 0;
        for (int k = 0; k < 128; ++k) want += (double)A[k * 64 + m] * B[k * 64 + n];
        const int lane = m + (n >= 32 ? 64 : 0), col = n % 32;
        const double got = D[lane * 64 + col];
        err = fmax(err, fabs(got - want));
        if (fabs(got - want) > 1e-2 && shown++ < 4) {
          // find where `want` appears
          int fl = -1, fc = -1;
          for (int l = 0; l < 128 && fl < 0; ++l) for (int c = 0; c < 64; ++c) if (fabs(D[l * 64 + c] - want) < 1e-3) { fl = l; fc = c; break; }
          printf("  m=%d n=%d want %.4f got %.4f (found at lane %d col %d)\n", m, n, want, got, fl, fc);
        }
      }
    printf("variant %d (%s): %s max err %g\n", variant, variant == 2 ? "K-major" : variant ? "MN lbo=512 sbo=8K" : "MN lbo=8K sbo=512", cudaGetErrorString(e), err);
    printf("  nonzero cols per lane:");
    for (int l = 0; l < 128; ++l) { int nz = 0; for (int c = 0; c < 64; ++c) nz += D[l * 64 + c] != 0.f; printf(" %d", nz); }
    printf("\n");
    // locate a few wanted values anywhere
    for (int t = 0; t < 6; ++t) {
      const int m = (t * 13) % 64, n = (t * 29) % 64;
      double want = 0;
      for (int k = 0; k < 128; ++k) want += (double)A[k * 64 + m] * B[k * 64 + n];
      printf("  want(m=%d,n=%d)=%.4f at:", m, n, want);
      for (int l = 0; l < 128; ++l) for (int c = 0; c < 64; ++c) if (fabs(D[l * 64 + c] - want) < 1e-3) printf(" (%d,%d)", l, c);
      printf("\n");
    }
  }
  return 0;
}

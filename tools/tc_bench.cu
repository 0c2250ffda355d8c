// tcgen05 kind::tf32 issue-rate microbenchmark: cycles per MMA for
// M (128 or 64) x N x K=8 with A/B in shared memory (SS) or A in TMEM, K-major,
// SW128 or SW64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/tc_bench.cu -o tools/tc_bench && ./tools/tc_bench
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
DEVI u64 sdesc(u32 saddr, int sw) {  // sw: 128 or 64
  const u64 sbo = sw == 128 ? 1024 : 512, lt = sw == 128 ? 2 : 4;
  return (u64)((saddr & 0x3FFFFu) >> 4) | ((u64)1 << 16) | ((sbo >> 4) << 32) | ((u64)1 << 46) | (lt << 61);
}

__global__ void bench(int n, int sw, int iters, long long* out, int a_tmem, int warp_issue, int fast, int mdim) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((unsigned long long)smem_raw + 1023) & ~1023ull);
  u64* bar = (u64*)(sm + 65536 + 131072);
  u32* tslot = (u32*)(bar + 1);
  for (int i = threadIdx.x; i < (65536 + 131072) / 4; i += blockDim.x) ((float*)sm)[i] = 1.0f;
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_addr(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = *tslot;
  if (warp_issue ? threadIdx.x < 32 : threadIdx.x == 0) {
    const u32 idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(n >> 3) << 17) | ((u32)(mdim >> 4) << 24);
    const u32 a = smem_addr(sm), b = smem_addr(sm + 65536);
    const int ksteps = sw == 128 ? 4 : 2;
    long long t0 = clock64();
    if (fast && !a_tmem) {
      const u64 ad0 = sdesc(a, sw), bd0 = sdesc(b, sw);
      for (int it = 0; it < iters; it += 4) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                       :: "r"(0u), "l"(ad0 + (sw == 128 ? 2 * ks : 2 * (ks & 1) + 256 * (ks >> 1))), "l"(bd0 + (sw == 128 ? 2 * ks : 2 * (ks & 1) + 256 * (ks >> 1))), "r"(idesc), "r"(1u) : "memory");
      }
    }
    if (fast && a_tmem) {  // A from TMEM columns 384.., D rotating over 4 column blocks
      const u64 bd0 = sdesc(b, sw);
      for (int it = 0; it < iters; it += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}"
                       :: "r"((u32)((j & 3) * 64)), "r"((u32)(384 + 8 * j)), "l"(bd0 + 2 * (j & 3)), "r"(idesc), "r"(1u) : "memory");
      }
    }
    for (int it = 0; it < (fast ? 0 : iters); ++it) {
      const int ks = it % ksteps;
      const int blk = (it / ksteps) % 4;  // rotate over 4 A tiles / 4 B tiles
      const u32 aa = a + blk * 16384 + ks * 32, bb = b + blk * n * 128 + ks * 32;
      u32 pred = 1;
      if (warp_issue) asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(pred));
      if (pred) {
      if (a_tmem) {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}"
                     :: "r"(tmem), "r"(tmem + 256 + ks * 8 + blk * 32), "l"(sdesc(bb, sw)), "r"(idesc), "r"(1u) : "memory");
      } else {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                     :: "r"(tmem), "l"(sdesc(aa, sw)), "l"(sdesc(bb, sw)), "r"(idesc), "r"(1u) : "memory");
      }
      }
      if (warp_issue) __syncwarp();
    }
    if (threadIdx.x == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_addr(bar)) : "memory");
    if (warp_issue) __syncwarp();
    while (!mbar_try(bar, 0)) { }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

int main() {
  long long* out;
  cudaMallocManaged(&out, 148 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  const int iters = 4096;
  for (int mdim : {128, 64})
  for (int at = 0; at < 2; ++at)
    for (int sw : {128, 64})
      for (int n : {64, 128, 256}) { if (at && (n == 256 || mdim == 64)) continue; {
        bench<<<148, 128, 200000>>>(n, sw, iters, out, at, 0, 1, mdim);
        printf("fast-unrolled M=%d ", mdim); fflush(stdout);
        cudaError_t e = cudaDeviceSynchronize();
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = out[i] > mx ? out[i] : mx;
        const double cyc = (double)mx / iters;
        printf("%s sw%-3d N=%-3d: %s  %.1f cycles/MMA  -> %.0f MAC/cycle/SM\n", at ? "A=TMEM" : "A=SMEM", sw, n,
               cudaGetErrorString(e), cyc, (double)mdim * n * 8 / cyc);
      } }
  return 0;
}

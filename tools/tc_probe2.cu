// tcgen05.commit arrival-count probe: does a barrier committed once get a
// second arrival from later commits to OTHER barriers?
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
DEVI bool wait_b(u64* b, u32 par) { long long t0 = clock64(); while (clock64() - t0 < 1000000000ll) if (mbar_try(b, par)) return true; return false; }
DEVI u64 sdesc(u32 saddr) { return (u64)((saddr & 0x3FFFFu) >> 4) | ((u64)1 << 16) | ((u64)(1024 >> 4) << 32) | ((u64)1 << 46) | ((u64)2 << 61); }
DEVI void commit(u64* b) { asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_addr(b)) : "memory"); }
__global__ void k(int* out, int variant) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((unsigned long long)smem_raw + 1023) & ~1023ull);
  u64* bar = (u64*)(sm + 24576);  // bar[0]=A bar[1]=W0 bar[2]=W1
  u32* tslot = (u32*)(bar + 4);
  for (int i = threadIdx.x; i < 24576 / 4; i += blockDim.x) ((float*)sm)[i] = 0.5f;
  if (threadIdx.x == 0) { for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" :: "r"(smem_addr(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = *tslot;
  if (threadIdx.x == 0) {
    const u32 idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(64 >> 3) << 17) | ((u32)(128 >> 4) << 24);
    for (int round = 0; round < 2; ++round) {
      for (int ks = 0; ks < 4; ++ks)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                     :: "r"(tmem), "l"(sdesc(smem_addr(sm) + ks * 32)), "l"(sdesc(smem_addr(sm + 16384) + ks * 32)), "r"(idesc), "r"(1u) : "memory");
      commit(&bar[0]);
      if (variant == 0 || round == 0) commit(&bar[1 + round]);
      out[round * 4 + 0] = wait_b(&bar[0], round & 1);
      if (variant == 0 || round == 0) out[round * 4 + 1] = wait_b(&bar[1 + round], 0);
      out[round * 4 + 2] = mbar_try(&bar[1], 0);  // W0 phase-0 completed and not twice
      out[round * 4 + 3] = mbar_try(&bar[1], 1);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tmem));
}
int main() {
  int* o; cudaMallocManaged(&o, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 30000);
  for (int v = 0; v < 2; ++v) {
    for (int i = 0; i < 8; ++i) o[i] = -1;
    k<<<1, 128, 30000>>>(o, v);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s  round0: A=%d W=%d W0par0=%d W0par1=%d | round1: A=%d W=%d W0par0=%d W0par1=%d\n", v,
           cudaGetErrorString(e), o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
  }
}

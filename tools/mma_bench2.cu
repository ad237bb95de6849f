// tcgen05 commit / completion-latency microbenchmark (sm_100a): groups of G MMAs
// (TS f16 M128 N16 K16), commit after each group; WAIT=1 waits for the group's
// completion (round trip), WAIT=0 only commits.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long sdesc(unsigned a, unsigned sbo) {
  return (unsigned long long)((a >> 4) & 0x3FFFu) | ((unsigned long long)(128u >> 4) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

template <int G, int WAIT, int SS>
__global__ void bench(int groups, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned tslot;
  __shared__ __align__(8) unsigned long long bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float*)sm)[i] = 0.001f * (i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = tslot;
  if (threadIdx.x == 0) {
    const unsigned idesc = SS ? ((1u << 4) | (2u << 7) | (2u << 10) | (8u << 17) | (8u << 24))
                              : ((1u << 4) | (2u << 17) | (8u << 24));
    const unsigned long long da = sdesc(saddr(sm), 512), db = sdesc(saddr(sm + 32768), 1024);
    unsigned phase = 0;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (SS)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + 256u), "l"(da + 16 * (i & 1)), "l"(db + 16 * (i & 1)), "r"(idesc), "r"((unsigned)(i > 0)));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem + 256u), "r"(tmem + (unsigned)((i & 3) * 8)), "l"(db + 16 * (i & 3)), "r"(idesc), "r"((unsigned)(i > 0)));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)));
      if (WAIT) {
        unsigned ok = 0;
        while (!ok)
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(saddr(&bar)), "r"(phase));
        phase ^= 1;
      }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int G, int WAIT, int SS>
void run() {
  long long* d;
  cudaMalloc(&d, 16);
  auto k = bench<G, WAIT, SS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  const int groups = 256;
  k<<<148, 128, 120 * 1024>>>(groups, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%s G=%2d wait=%d: %.1f cyc/group, %.1f cyc/mma %s\n", SS ? "SS tf32 N64" : "TS f16 N16 ", G, WAIT,
         (double)h / groups, (double)h / groups / G, e ? cudaGetErrorString(e) : "");
  cudaFree(d);
}

int main() {
  run<1, 0, 0>(); run<2, 0, 0>(); run<8, 0, 0>(); run<32, 0, 0>();
  run<1, 1, 0>(); run<2, 1, 0>(); run<8, 1, 0>(); run<32, 1, 0>();
  run<6, 0, 1>(); run<6, 1, 1>(); run<3, 1, 1>();
  return 0;
}

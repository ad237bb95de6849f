// tcgen05.mma issue/throughput microbenchmark for the K1-TC shapes (sm_100a).
// One CTA per SM; one thread issues R back-to-back MMAs, then commit + wait.
// Reports cycles per MMA for SS (A,B in SMEM) and TS (A in TMEM) forms.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long sdesc(unsigned a, unsigned sbo) {
  return (unsigned long long)((a >> 4) & 0x3FFFu) | ((unsigned long long)(128u >> 4) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

template <int KIND, int TS>  // KIND 0 = tf32, 1 = f16
__global__ void bench(int n_mma, int N, int alt, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned tslot;
  __shared__ __align__(8) unsigned long long bar;
  __shared__ __align__(8) unsigned long long bar2;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float*)sm)[i] = 0.001f * (i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(saddr(&bar2)));
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
    const unsigned fmt = KIND == 0 ? 2u : 0u;
    const unsigned idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((unsigned)(N >> 3) << 17) | (8u << 24);
    const unsigned long long da = sdesc(saddr(sm), 512), db = sdesc(saddr(sm + 32768), 512);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const unsigned d = tmem + 256u + (alt == 1 ? (unsigned)((i & 1) * 64) : 0u);
      const unsigned acc = i > 1;
      if (TS) {
        const unsigned a = tmem + (unsigned)((i & 3) * 8);
        if (KIND == 0)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(db + 16 * (i & 3)), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(db + 16 * (i & 3)), "r"(idesc), "r"(acc));
      } else {
        if (KIND == 0)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(da + 16 * (i & 1)), "l"(db + 16 * (i & 1)), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(da + 16 * (i & 1)), "l"(db + 16 * (i & 1)), "r"(idesc), "r"(acc));
      }
      if (alt >= 2 && (i % alt) == alt - 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar2)));
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)));
    unsigned ok = 0;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(saddr(&bar)));
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int KIND, int TS>
void run(const char* name, int N, int alt) {
  long long* d;
  cudaMalloc(&d, 16);
  auto k = bench<KIND, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  for (int n_mma : {64, 1024}) {
    k<<<148, 128, 120 * 1024>>>(n_mma, N, alt, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-28s N=%3d alt=%d n=%5d: issue %.1f cyc/mma, total %.1f cyc/mma %s\n", name, N, alt, n_mma,
           (double)h[0] / n_mma, (double)h[1] / n_mma, e ? cudaGetErrorString(e) : "");
  }
  cudaFree(d);
}

int main() {
  run<1, 1>("TS f16 N16 commit/1", 16, 2 - 1 + 1);
  run<1, 1>("TS f16 N16 commit/2", 16, 2);
  run<1, 1>("TS f16 N16 commit/4", 16, 4);
  run<1, 1>("TS f16 N16 commit/8", 16, 8);
  run<0, 0>("SS tf32 N64 commit/3", 64, 3);
  run<0, 0>("SS tf32 N64 commit/6", 64, 6);
  run<0, 0>("SS tf32 M128 K8", 64, 0);
  run<0, 0>("SS tf32 M128 K8", 64, 1);
  run<0, 0>("SS tf32 M128 K8", 128, 0);
  run<0, 0>("SS tf32 M128 K8", 256, 0);
  run<0, 1>("TS tf32 M128 K8", 16, 0);
  run<0, 1>("TS tf32 M128 K8", 64, 0);
  run<1, 1>("TS f16 M128 K16", 16, 0);
  run<1, 1>("TS f16 M128 K16", 16, 1);
  run<1, 1>("TS f16 M128 K16", 64, 0);
  run<1, 1>("TS f16 M128 K16", 256, 0);
  run<1, 0>("SS f16 M128 K16", 16, 0);
  run<1, 0>("SS f16 M128 K16", 64, 0);
  run<1, 0>("SS f16 M128 K16", 256, 0);
  return 0;
}

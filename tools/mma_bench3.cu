// tcgen05 issue-rate microbenchmark, part 3 (sm_100a): cta_group::2 (M = 256
// over a CTA pair) versus cta_group::1 (M = 128), and two concurrent issuing
// threads on one SM. R MMAs per issuer, a commit every 8, final wait.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_bench3 tools/mma_bench3.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long sdesc(unsigned a, unsigned sbo) {
  return (unsigned long long)((a >> 4) & 0x3FFFu) | ((unsigned long long)(128u >> 4) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ unsigned ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int R = 2048;

__device__ volatile int g_stop;

template <int CG, int TS, int N, int NISS, int BG = 0>
__device__ void body(long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned tslot;
  __shared__ __align__(8) unsigned long long bar[6];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((float*)sm)[i] = 0.001f * (i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[1])));
    for (int q = 2; q < 6; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = tslot;
  const bool issuer = (CG == 1 || ctarank() == 0) && (threadIdx.x % 32 == 0) && warp < NISS;
  if (issuer) {
    const int w = warp;
    const unsigned m = CG == 2 ? 256u : 128u;
    const unsigned idesc = (1u << 4) | ((unsigned)(N >> 3) << 17) | ((m >> 4) << 24);
    const unsigned long long da = sdesc(saddr(sm), 512), db = sdesc(saddr(sm + 32768), 1024);
    const unsigned dcol = 256u + 64u * (unsigned)w;
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const unsigned acc = (i & 7) != 0;
      const unsigned d = tmem + dcol;
      if (TS) {
        const unsigned a = tmem + (unsigned)((i & 3) * 8) + 32u * (unsigned)w;
        if (CG == 1)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(db + 16 * (i & 3)), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a), "l"(db + 16 * (i & 3)), "r"(idesc), "r"(acc));
      } else {
        if (CG == 1)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(da + 16 * (i & 1)), "l"(db + 16 * (i & 1)), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(da + 16 * (i & 1)), "l"(db + 16 * (i & 1)), "r"(idesc), "r"(acc));
      }
      if ((i & 7) == 7 && i != R - 1) {
        // mid-stream commits (to a barrier nobody waits on), as a real pipeline does
        if (CG == 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar[1])));
        else
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(saddr(&bar[1])), "h"((unsigned short)3));
      }
    }
    long long t1 = clock64();
    const unsigned fin = saddr(&bar[w == 0 ? 0 : 1 + w]);
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(fin));
    else
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(fin), "h"((unsigned short)(w == 0 ? 3 : 1)));
    unsigned ok = 0;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(fin));
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[2 * w] = t1 - t0;
      out[2 * w + 1] = t2 - t0;
    }
  } else if (BG && warp >= 4) {
    // epilogue-like TMEM traffic: 64 columns ld, 64 columns st, per iteration
    const unsigned lanes = (unsigned)(32 * (warp & 3)) << 16;
    const unsigned base = tmem + 128u + 64u * (unsigned)((warp - 4) >> 2 & 1) + lanes;
    unsigned v[32];
    for (int it = 0; it < 1200; ++it) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                     "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(base));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 32; ++j) v[j] += it;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   :: "r"(base), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  } else if (CG == 2 && ctarank() == 1 && threadIdx.x == 0) {
    unsigned ok = 0;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(saddr(&bar[0])));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) cluster_sync();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int TS, int N, int NISS>
__global__ void k1(long long* out) { body<1, TS, N, NISS>(out); }
template <int TS, int N, int NISS>
__global__ void k1bg(long long* out) { body<1, TS, N, NISS, 1>(out); }
template <int TS, int N, int NISS>
__global__ void __cluster_dims__(2, 1, 1) k2(long long* out) { body<2, TS, N, NISS>(out); }

template <class K>
void run(K k, const char* name, int niss, int threads = 128) {
  long long* d;
  cudaMalloc(&d, 64);
  cudaMemset(d, 0, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  k<<<148, threads, 120 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  double worst = 0;
  for (int w = 0; w < niss; ++w) worst = h[2 * w + 1] > worst ? h[2 * w + 1] : worst;
  printf("%-34s issue %.1f cyc/mma/issuer, total %.1f cyc/mma per SM-or-pair %s\n", name,
         (double)h[0] / R, worst / (R * niss), e ? cudaGetErrorString(e) : "");
  fflush(stdout);
  cudaFree(d);
}

int main() {
  run(k1<1, 32, 2>, "cg1 TS f16 M128 N32 K16 x2 issuers", 2);
  run(k1bg<1, 32, 2>, "  + 8 warps TMEM ld/st traffic", 2, 384);
  run(k1<0, 64, 2>, "cg1 SS f16 M128 N64 K16 x2 issuers", 2);
  run(k1bg<0, 64, 2>, "  + 8 warps TMEM ld/st traffic", 2, 384);
  run(k1<1, 32, 1>, "cg1 TS f16 M128 N32 K16 x1", 1);
  run(k1bg<1, 32, 1>, "  + 8 warps TMEM ld/st traffic", 1, 384);
  return 0;
}

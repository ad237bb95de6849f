// Layout check for tcgen05.mma.cta_group::2 (M = 256 over a CTA pair), sm_100a:
// which CTA's shared memory supplies which rows of B, and where D lands.
// A (256 x 16 FP16, K-major): CTA r holds rows 128r..128r+127 (SMEM, or TMEM
// for the TS form). B (N x 16): CTA r holds rows (N/2) r .. (N/2)(r+1)-1.
// D is read back from each CTA's TMEM and compared with a host GEMM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/cg2_check tools/cg2_check.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
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
// K-major no-swizzle FP16 tile with 16 K columns: 8-row groups of 256 B, K chunks 128 B apart
__device__ __forceinline__ int off(int r, int k) { return (r >> 3) * 128 + (k >> 3) * 64 + (r & 7) * 8 + (k & 7); }

__host__ __device__ inline float aval(int r, int k) { return (float)((r * 7 + k * 3) % 11 - 5) * 0.25f; }
__host__ __device__ inline float bval(int n, int k) { return (float)((n * 5 + k * 13) % 9 - 4) * 0.5f; }

template <int TS, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) kern(float* out) {
  __shared__ __align__(1024) __half As[128 * 16];
  __shared__ __align__(1024) __half Bs[(N / 2) * 16];
  __shared__ unsigned tslot;
  __shared__ __align__(8) unsigned long long bar;
  const unsigned rank = ctarank();
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < 128 * 16; i += 128) {
    const int r = i / 16, k = i % 16;
    As[off(r, k)] = __float2half(aval(128 * rank + r, k));
  }
  for (int i = tid; i < (N / 2) * 16; i += 128) {
    const int n = i / 16, k = i % 16;
    Bs[off(n, k)] = __float2half(bval((N / 2) * rank + n, k));
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(saddr(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = tslot;
  if (TS) {
    // A rows into this CTA's TMEM columns 0..7 (FP16x2 along K), lane = row
    unsigned v[8];
    const int r = tid;
    for (int c = 0; c < 8; ++c) {
      __half2 h = __halves2half2(__float2half(aval(128 * rank + r, 2 * c)), __float2half(aval(128 * rank + r, 2 * c + 1)));
      v[c] = *reinterpret_cast<unsigned*>(&h);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + ((unsigned)(32 * warp) << 16)),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (rank == 0 && tid == 0) {
    const unsigned idesc = (1u << 4) | ((unsigned)(N >> 3) << 17) | ((256u >> 4) << 24);
    const unsigned long long da = sdesc(saddr(As), 256), db = sdesc(saddr(Bs), 256);
    const unsigned d = tmem + 128u;
    if (TS)
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(tmem), "l"(db), "r"(idesc), "r"(0u));
    else
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(da), "l"(db), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(saddr(&bar)), "h"((unsigned short)3));
  }
  {
    unsigned ok = 0;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(saddr(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 8) {
    unsigned v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + 128u + (unsigned)c0 + ((unsigned)(32 * warp) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[(size_t)(rank * 128 + 32 * warp + lane) * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

template <int TS, int N>
int check(const char* name) {
  float* d;
  cudaMalloc(&d, 256 * N * 4);
  cudaMemset(d, 0xff, 256 * N * 4);
  kern<TS, N><<<2, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  float* h = (float*)malloc(256 * N * 4);
  cudaMemcpy(h, d, 256 * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < N; ++n) {
      float ref = 0;
      for (int k = 0; k < 16; ++k) ref += aval(m, k) * bval(n, k);
      if (h[m * N + n] != ref) {
        if (bad < 4) printf("  %s mismatch D[%d][%d] = %g, want %g\n", name, m, n, h[m * N + n], ref);
        ++bad;
      }
    }
  printf("%s: %s, %d mismatches of %d %s\n", name, bad ? "FAIL" : "ok", bad, 256 * N, e ? cudaGetErrorString(e) : "");
  fflush(stdout);
  free(h);
  cudaFree(d);
  return bad;
}

int main() {
  int bad = 0;
  bad += check<0, 64>("cg2 SS M256 N64");
  bad += check<1, 32>("cg2 TS M256 N32");
  bad += check<0, 32>("cg2 SS M256 N32");
  return bad ? 1 : 0;
}

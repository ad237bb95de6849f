// Layout check for an MN-major FP16 A operand in SMEM (no swizzle), sm_100a:
// D[128 x 32] = A[128 x 16] . B[32 x 16]^T with A written "MN-major" (for each
// K index, 8 consecutive M elements in 16 B), as a row-owning epilogue thread
// would store P^T, and B K-major. Tries the two LBO/SBO assignments.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mnmajor_check tools/mnmajor_check.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long sdesc(unsigned a, unsigned lbo, unsigned sbo) {
  return (unsigned long long)((a >> 4) & 0x3FFFu) | ((unsigned long long)((lbo >> 4) & 0x3FFFu) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__host__ __device__ inline float aval(int m, int k) { return (float)((m * 7 + k * 3) % 11 - 5) * 0.25f; }
__host__ __device__ inline float bval(int n, int k) { return (float)((n * 5 + k * 13) % 9 - 4) * 0.5f; }

// A element (m, k): core matrix (m >> 3, k >> 3) at mb * 128 + kb * 2048 bytes,
// inside it K-row (k & 7) of 16 B holding m & 7
__device__ __forceinline__ int aoff(int m, int k, int kmajor) {
  if (kmajor) return (m >> 3) * 128 + (k >> 3) * 64 + (m & 7) * 8 + (k & 7);  // control
  return ((m >> 3) * 128 + (k >> 3) * 2048) / 2 + (k & 7) * 8 + (m & 7);
}
// B K-major: (n, k) -> 8-row groups of 256 B, K chunks 128 B apart
__device__ __forceinline__ int boff(int n, int k) { return (n >> 3) * 128 + (k >> 3) * 64 + (n & 7) * 8 + (k & 7); }

__global__ void kern(int variant, float* out) {
  __shared__ __align__(1024) __half As[128 * 16 + 1024];
  __shared__ __align__(1024) __half Bs[32 * 16];
  __shared__ unsigned tslot;
  __shared__ __align__(8) unsigned long long bar;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int kmajor = variant == 9;
  for (int i = tid; i < 128 * 16; i += 128) As[aoff(i / 16, i % 16, kmajor)] = __float2half(aval(i / 16, i % 16));
  for (int i = tid; i < 32 * 16; i += 128) Bs[boff(i / 16, i % 16)] = __float2half(bval(i / 16, i % 16));
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(saddr(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = tslot;
  if (tid == 0) {
    // a_major (bit 15) = MN-major
    const unsigned idesc = (1u << 4) | (kmajor ? 0u : (1u << 15)) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    const unsigned lbos[] = {128u, 2048u, 128u, 2048u, 256u};
    const unsigned sbos[] = {2048u, 128u, 1024u, 256u, 2048u};
    unsigned lbo = kmajor ? 128u : lbos[variant], sbo = kmajor ? 256u : sbos[variant];
    const unsigned long long da = sdesc(saddr(As), lbo, sbo);
    const unsigned long long db = sdesc(saddr(Bs), 128u, 256u);
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)));
  }
  unsigned ok = 0;
  while (!ok)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(saddr(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 32; c0 += 8) {
    unsigned v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + (unsigned)c0 + ((unsigned)(32 * warp) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[(32 * warp + lane) * 32 + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  }
}

int main(int argc, char** argv) {
  const int variant = atoi(argv[1]);
  float* d;
  cudaMalloc(&d, 128 * 32 * 4);
  static float h[128 * 32];
  cudaMemset(d, 0, 128 * 32 * 4);
  kern<<<1, 128>>>(variant, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      float ref = 0;
      for (int k = 0; k < 16; ++k) ref += aval(m, k) * bval(n, k);
      bad += h[m * 32 + n] != ref;
    }
  printf("variant %d: %d mismatches %s\n", variant, bad, e ? cudaGetErrorString(e) : "");
  return bad != 0;
}

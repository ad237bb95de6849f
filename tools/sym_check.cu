// Is the tensor-core distance GEMM bitwise symmetric for a point set against
// itself? S'[i][j] = a_i . b_j over K = 3D + 4 FP16 hi/lo terms (kind::f16,
// FP32 accumulate, 2 MMAs of K = 16). Layout 0 = the K1-TC layout
// [c_hi | c_hi | c_lo | n_hi n_lo 1 1] / [2c_hi | 2c_lo | 2c_hi | -1 -1 -m_hi -m_lo];
// layout 1 = "paired": the two cross terms of each coordinate and the two
// halves of each norm term sit in adjacent K slots, so swapping i and j only
// swaps adjacent products. Counts asymmetric entries of S'.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/sym_check tools/sym_check.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <vector>

constexpr int D = 8, KH = 32, NP = 128;

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long sdesc(unsigned a, unsigned lbo, unsigned sbo) {
  return (unsigned long long)((a >> 4) & 0x3FFFu) | ((unsigned long long)((lbo >> 4) & 0x3FFFu) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__host__ __device__ inline int koff(int r, int k) { return (r >> 3) * (KH * 8) + (k >> 3) * 64 + (r & 7) * 8 + (k & 7); }

__global__ void kern(const __half* A, const __half* B, float* out) {
  __shared__ __align__(1024) __half As[NP * KH];
  __shared__ __align__(1024) __half Bs[NP * KH];
  __shared__ unsigned tslot;
  __shared__ __align__(8) unsigned long long bar;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < NP * KH; i += 128) { As[i] = A[i]; Bs[i] = B[i]; }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(saddr(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = tslot;
  if (tid == 0) {
    const unsigned idesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    const unsigned long long da = sdesc(saddr(As), 128, KH * 16), db = sdesc(saddr(Bs), 128, KH * 16);
    for (int kk = 0; kk < KH / 16; ++kk)
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem), "l"(da + 16 * kk), "l"(db + 16 * kk), "r"(idesc), "r"((unsigned)(kk > 0)));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)));
  }
  unsigned ok = 0;
  while (!ok)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(saddr(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 128; c0 += 8) {
    unsigned v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + (unsigned)c0 + ((unsigned)(32 * warp) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[(32 * warp + lane) * 128 + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  }
}

static void split(double v, __half& hi, __half& lo) {
  hi = __double2half(v);
  lo = __double2half(v - (double)__half2float(hi));
}

int main() {
  srand(7);
  std::vector<double> c(NP * D), nn(NP);
  for (int i = 0; i < NP; ++i) {
    nn[i] = 0;
    for (int d = 0; d < D; ++d) {
      c[i * D + d] = ((double)rand() / RAND_MAX - 0.5) * 2.4;
      nn[i] += c[i * D + d] * c[i * D + d];
    }
  }
  __half *dA, *dB;
  float* dO;
  cudaMalloc(&dA, NP * KH * 2);
  cudaMalloc(&dB, NP * KH * 2);
  cudaMalloc(&dO, NP * NP * 4);
  const __half one = __float2half(1.f), mone = __float2half(-1.f), zero = __float2half(0.f);
  for (int layout = 0; layout < 2; ++layout) {
    std::vector<__half> A(NP * KH, zero), B(NP * KH, zero);
    for (int i = 0; i < NP; ++i) {
      __half ch[D], cl[D], c2h[D], c2l[D], nh, nl;
      for (int d = 0; d < D; ++d) {
        split(c[i * D + d], ch[d], cl[d]);
        split(2.0 * c[i * D + d], c2h[d], c2l[d]);
      }
      split(nn[i], nh, nl);
      const __half mnh = __hneg(nh), mnl = __hneg(nl);
      auto put = [&](int k, __half a, __half b) {
        A[koff(i, k)] = a;
        B[koff(i, k)] = b;
      };
      if (layout == 0) {
        for (int d = 0; d < D; ++d) {
          put(d, ch[d], c2h[d]);
          put(D + d, ch[d], c2l[d]);
          put(2 * D + d, cl[d], c2h[d]);
        }
        put(3 * D, nh, mone);
        put(3 * D + 1, nl, mone);
        put(3 * D + 2, one, mnh);
        put(3 * D + 3, one, mnl);
      } else {
        for (int d = 0; d < D; ++d) {
          put(d, ch[d], c2h[d]);
          put(D + 2 * d, ch[d], c2l[d]);      // (i, j): c_hi^i * 2c_lo^j
          put(D + 2 * d + 1, cl[d], c2h[d]);  // (i, j): c_lo^i * 2c_hi^j; (j, i) swaps the pair
        }
        put(3 * D, nh, mone);
        put(3 * D + 1, one, mnh);
        put(3 * D + 2, nl, mone);
        put(3 * D + 3, one, mnl);
      }
    }
    cudaMemcpy(dA, A.data(), NP * KH * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), NP * KH * 2, cudaMemcpyHostToDevice);
    kern<<<1, 128>>>(dA, dB, dO);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> S(NP * NP);
    cudaMemcpy(S.data(), dO, NP * NP * 4, cudaMemcpyDeviceToHost);
    int asym = 0;
    double maxerr = 0;
    for (int i = 0; i < NP; ++i)
      for (int j = 0; j < NP; ++j) {
        if (S[i * NP + j] != S[j * NP + i]) ++asym;
        double r2 = 0;
        for (int d = 0; d < D; ++d) r2 += (c[i * D + d] - c[j * D + d]) * (c[i * D + d] - c[j * D + d]);
        maxerr = fmax(maxerr, fabs(S[i * NP + j] + r2));
      }
    printf("layout %d: %d of %d entries asymmetric, max |S' + r^2| = %.3g %s\n", layout, asym, NP * NP, maxerr,
           e ? cudaGetErrorString(e) : "");
  }
  return 0;
}

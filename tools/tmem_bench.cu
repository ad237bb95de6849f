// TMEM load / store throughput microbenchmark (sm_100a): W warps per SM each
// loop tcgen05.ld (and/or st) over their lane quarter; reports bytes/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

#define R8(a, o) "=r"(a[o + 0]), "=r"(a[o + 1]), "=r"(a[o + 2]), "=r"(a[o + 3]), "=r"(a[o + 4]), "=r"(a[o + 5]), "=r"(a[o + 6]), "=r"(a[o + 7])
#define W8(a, o) "r"(a[o + 0]), "r"(a[o + 1]), "r"(a[o + 2]), "r"(a[o + 3]), "r"(a[o + 4]), "r"(a[o + 5]), "r"(a[o + 6]), "r"(a[o + 7])

constexpr int IT = 2048;

// MODE 0: ld 32x32b.x32 (x2 per iter, one wait); 1: st 32x32b.x32 (x2, one wait);
// 2: ld 16x256b.x8 (x2, one wait); 3: ld + st (epilogue-like)
template <int MODE, int COLS = 512>
__global__ void kern(long long* out, unsigned* sink) {
  __shared__ unsigned tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tslot)), "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = tslot;
  const unsigned lanes = (unsigned)(32 * (warp & 3)) << 16;
  const unsigned col = COLS == 512 ? 128u * (unsigned)((warp >> 2) & 3) : 64u * (unsigned)((warp >> 2) & 1);
  unsigned v[64];
  for (int i = 0; i < 64; ++i) v[i] = i * threadIdx.x;
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
    const unsigned a = tmem + lanes + col + 64u * (unsigned)(it & 1);
    if (MODE == 0 || MODE == 3) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 0), R8(v, 8), R8(v, 16), R8(v, 24) : "r"(a));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 32), R8(v, 40), R8(v, 48), R8(v, 56) : "r"(a + 32u));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= v[0] ^ v[31] ^ v[32] ^ v[63];  // fixed indices: a dynamic index puts v[] in local memory
    }
    if (MODE == 4) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
                   "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
                   : R8(v, 0), R8(v, 8), R8(v, 16), R8(v, 24), R8(v, 32), R8(v, 40), R8(v, 48), R8(v, 56) : "r"(a));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= v[0] ^ v[31] ^ v[32] ^ v[63];  // fixed indices: a dynamic index puts v[] in local memory
    }
    if (MODE == 5) {  // no wait between iterations: 4 loads in flight, one wait per 2 iterations
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 0), R8(v, 8), R8(v, 16), R8(v, 24) : "r"(a));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 32), R8(v, 40), R8(v, 48), R8(v, 56) : "r"(a + 32u));
      if (it & 1) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= v[0] ^ v[31] ^ v[32] ^ v[63];  // fixed indices: a dynamic index puts v[] in local memory
    }
    if (MODE == 2) {
      // 16x256b: 16 lanes x 256 bits per "row"; .x8 -> 32 registers per thread
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 0), R8(v, 8), R8(v, 16), R8(v, 24) : "r"(a));
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 32), R8(v, 40), R8(v, 48), R8(v, 56) : "r"(a + 32u));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= v[0] ^ v[31] ^ v[32] ^ v[63];  // fixed indices: a dynamic index puts v[] in local memory
    }
    if (MODE == 8) {  // 16x128b.x16: 32 registers per thread per load
      asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 0), R8(v, 8), R8(v, 16), R8(v, 24) : "r"(a));
      asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 32), R8(v, 40), R8(v, 48), R8(v, 56) : "r"(a + 32u));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= v[0] ^ v[31] ^ v[32] ^ v[63];
    }
    if (MODE == 9) {  // 16x64b.x32: 32 registers per thread per load
      asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 0), R8(v, 8), R8(v, 16), R8(v, 24) : "r"(a));
      asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : R8(v, 32), R8(v, 40), R8(v, 48), R8(v, 56) : "r"(a + 32u));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= v[0] ^ v[31] ^ v[32] ^ v[63];
    }
    if (MODE == 10) {  // 16x256b.x4 (the symmetric kernel's shape): 16 registers per load, 4 loads
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : R8(v, 0), R8(v, 8) : "r"(a));
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : R8(v, 16), R8(v, 24) : "r"(a + 16u));
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : R8(v, 32), R8(v, 40) : "r"(a + 32u));
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : R8(v, 48), R8(v, 56) : "r"(a + 48u));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= v[0] ^ v[31] ^ v[32] ^ v[63];
    }
    if (MODE == 1 || MODE == 3) {
      v[0] += it;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   ::"r"(a), W8(v, 0), W8(v, 8), W8(v, 16), W8(v, 24) : "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   ::"r"(a + 32u), W8(v, 32), W8(v, 40), W8(v, 48), W8(v, 56) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ v[5];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(COLS));
  }
}

template <int MODE>
void run(const char* name, int warps) {
  long long* d;
  unsigned* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  kern<MODE><<<148, 32 * warps>>>(d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)IT * warps * 32 * 64 * 4 * (MODE == 3 ? 2 : 1);
  printf("%-30s warps=%2d: %.1f B/clk/SM (%.0f cyc per iteration) %s\n", name, warps, bytes / h,
         (double)h / IT, e ? cudaGetErrorString(e) : "");
  fflush(stdout);
  cudaFree(d);
  cudaFree(sink);
}

// two co-resident CTAs per SM, 256 TMEM columns each: is the ld limit per SM or per CTA?
void run_two(int warps) {
  long long* d;
  unsigned* sink;
  cudaMalloc(&d, 296 * 8);
  cudaMalloc(&sink, 296 * 1024 * 4);
  kern<0, 256><<<296, 32 * warps>>>(d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)IT * warps * 32 * 64 * 4;
  printf("2 CTAs/SM x %d warps: %.1f B/clk per CTA (x2 per SM if co-resident) %s\n", warps, bytes / h,
         e ? cudaGetErrorString(e) : "");
  fflush(stdout);
}

// same total tcgen05.ld work, 1 CTA/SM x 8 warps vs 2 CTAs/SM x 4 warps: wall time by events
void run_total() {
  long long* d;
  unsigned* sink;
  cudaMalloc(&d, 296 * 8);
  cudaMalloc(&sink, 296 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    float ms1, ms2;
    cudaEventRecord(e0);
    kern<0, 512><<<148, 256>>>(d, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0);
    kern<0, 256><<<296, 128>>>(d, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms2, e0, e1);
    const double bytes = (double)IT * 8 * 32 * 64 * 4 * 148;
    printf("1 CTA/SM x 8 warps: %.3f ms (%.1f B/clk/SM at 1965 MHz); 2 CTAs/SM x 4 warps: %.3f ms (%.1f B/clk/SM)\n",
           ms1, bytes / (ms1 * 1e-3 * 1.965e9) / 148, ms2, bytes / (ms2 * 1e-3 * 1.965e9) / 148);
  }
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  for (int w : {4, 8, 16}) {
    if (mode == 0) run<0>("ld 32x32b.x32 x2 (64 cols)", w);
    if (mode == 1) run<1>("st 32x32b.x32 x2 (64 cols)", w);
    if (mode == 2 && w <= 8) run<2>("ld 16x256b.x8 x2", w);
    if (mode == 3) run<3>("ld+st 32x32b (64 cols)", w);
    if (mode == 4) run<4>("ld 32x32b.x64 (64 cols)", w);
    if (mode == 5) run<5>("ld x32 x2, wait every 2nd", w);
    if (mode == 6 && w <= 8) run_two(w);
    if (mode == 7 && w == 4) run_total();
    if (mode == 8 && w <= 8) run<8>("ld 16x128b.x16 x2", w);
    if (mode == 9 && w <= 8) run<9>("ld 16x64b.x32 x2", w);
    if (mode == 10 && w <= 8) run<10>("ld 16x256b.x4 x4", w);
  }
  return 0;
}

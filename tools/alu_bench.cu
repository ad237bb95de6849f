// SIMT pipe-throughput microbenchmark for the K1-TC epilogue (sm_100a):
// MUFU.EX2, FFMA, the FP16 hi/lo split and the whole per-entry epilogue
// sequence, with W warps per SM and 16 independent chains per thread.
// Reports SM-wide throughput in operations (entries) per clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/alu_bench tools/alu_bench.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 16;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void split(float x0, float x1, unsigned& hi, unsigned& lo) {
  unsigned h, l;
  float f0, f1;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x1), "f"(x0));
  asm("{\n\t.reg .f16 a, b;\n\tmov.b32 {a, b}, %2;\n\tcvt.f32.f16 %0, a;\n\tcvt.f32.f16 %1, b;\n\t}"
      : "=f"(f0), "=f"(f1)
      : "r"(h));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(x1 - f1), "f"(x0 - f0));
  hi = h;
  lo = l;
}

// split through the mixed-precision FMA (FHFMA): lo = x - f32(hi) in one op
__device__ __forceinline__ void split_fh(float x0, float x1, unsigned& hi, unsigned& lo) {
  unsigned h, l;
  float l0, l1;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x1), "f"(x0));
  asm("{\n\t.reg .f16 a, b, m;\n\tmov.b32 {a, b}, %2;\n\tmov.b16 m, 0xBC00;\n\t"
      "fma.rn.f32.f16 %0, a, m, %3;\n\tfma.rn.f32.f16 %1, b, m, %4;\n\t}"
      : "=f"(l0), "=f"(l1)
      : "r"(h), "f"(x0), "f"(x1));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(l1), "f"(l0));
  hi = h;
  lo = l;
}

// split by truncation: hi = x with 10 mantissa bits (exact in FP16 for
// x >= 2^-14), lo = x - hi
__device__ __forceinline__ void split_tr(float x0, float x1, unsigned& hi, unsigned& lo) {
  unsigned h, l;
  const float h0 = __uint_as_float(__float_as_uint(x0) & 0xFFFFE000u);
  const float h1 = __uint_as_float(__float_as_uint(x1) & 0xFFFFE000u);
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(h1), "f"(h0));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(x1 - h1), "f"(x0 - h0));
  hi = h;
  lo = l;
}

// 2^x for x <= 0 on the FMA pipe: round-to-nearest range reduction, degree-5
// minimax-like polynomial on [-0.5, 0.5], exponent added with an integer op
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float n = t - 12582912.f;
  const float f = x - n;
  float p = 1.3333558e-3f;
  p = fmaf(p, f, 9.6181291e-3f);
  p = fmaf(p, f, 5.5504109e-2f);
  p = fmaf(p, f, 2.4022651e-1f);
  p = fmaf(p, f, 6.9314718e-1f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int MODE>
__global__ void bench(float seed, float* out, long long* cyc) {
  float v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = -0.001f * (threadIdx.x + c) * seed;
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    if (MODE == 0) {  // MUFU.EX2 only
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = ex2(v[c]) - 1.0f;
    } else if (MODE == 1) {  // FFMA only
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = fmaf(v[c], 0.999f, -0.001f);
    } else if (MODE == 2) {  // split only (per 2 entries)
#pragma unroll
      for (int c = 0; c < CH; c += 2) {
        unsigned h, l;
        split(v[c], v[c + 1], h, l);
        v[c] = __uint_as_float(h ^ l) - 0.5f;
        v[c + 1] = __uint_as_float(h) * 0.5f;
      }
    } else if (MODE == 3) {  // full entry: fmin, ex2, split
#pragma unroll
      for (int c = 0; c < CH; c += 2) {
        unsigned h, l;
        split(ex2(fminf(v[c], 0.f)), ex2(fminf(v[c + 1], 0.f)), h, l);
        acc += h ^ l;
        v[c] -= 0.01f;
        v[c + 1] -= 0.01f;
      }
    } else if (MODE == 5 || MODE == 6) {  // alternative splits only
#pragma unroll
      for (int c = 0; c < CH; c += 2) {
        unsigned h, l;
        if (MODE == 5) split_fh(v[c], v[c + 1], h, l);
        else split_tr(v[c], v[c + 1], h, l);
        v[c] = __uint_as_float(h ^ l) - 0.5f;
        v[c + 1] = __uint_as_float(h) * 0.5f;
      }
    } else if (MODE == 7 || MODE == 8) {  // full entry with the alternative splits
#pragma unroll
      for (int c = 0; c < CH; c += 2) {
        unsigned h, l;
        const float e0 = ex2(fminf(v[c], 0.f)), e1 = ex2(fminf(v[c + 1], 0.f));
        if (MODE == 7) split_fh(e0, e1, h, l);
        else split_tr(e0, e1, h, l);
        acc += h ^ l;
        v[c] -= 0.01f;
        v[c + 1] -= 0.01f;
      }
    } else if (MODE == 9) {  // F2FP pack only
#pragma unroll
      for (int c = 0; c < CH; c += 2) {
        unsigned h;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(v[c + 1]), "f"(v[c]));
        acc += h;
      }
    } else if (MODE == 10) {  // HADD2.F32 unpack only
#pragma unroll
      for (int c = 0; c < CH; c += 2) {
        float f0, f1;
        const unsigned h = __float_as_uint(v[c]) ^ acc;
        asm volatile("{\n\t.reg .f16 a, b;\n\tmov.b32 {a, b}, %2;\n\tcvt.f32.f16 %0, a;\n\tcvt.f32.f16 %1, b;\n\t}"
            : "=f"(f0), "=f"(f1) : "r"(h));
        v[c] = f0;
        v[c + 1] += f1;
      }
    } else if (MODE == 4) {  // polynomial exp2 only
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = ex2_poly(v[c]) - 1.0f;
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
  float* o;
  long long* c;
  cudaMalloc(&o, 148 * 1024 * 4);
  cudaMalloc(&c, 148 * 8);
  bench<MODE><<<148, 32 * warps>>>(1.0f, o, c);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)ITERS * CH * 32 * warps;
  printf("%-28s warps/SM=%2d: %.2f ops/clk/SM (%.1f cyc per warp-op per SMSP) %s\n", name, warps,
         ops / h, 4.0 * 32 * (double)h / ops, e ? cudaGetErrorString(e) : "");
  fflush(stdout);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  for (int w : {4, 8, 16}) run<0>("MUFU.EX2", w);
  for (int w : {4, 8}) run<1>("FFMA", w);
  for (int w : {4, 8}) run<2>("fp16 hi/lo split", w);
  for (int w : {4, 8, 16}) run<3>("fmin+ex2+split (entry)", w);
  for (int w : {4, 8}) run<4>("poly exp2", w);
  for (int w : {8, 16}) run<5>("split via FHFMA", w);
  for (int w : {8, 16}) run<6>("split via truncation", w);
  for (int w : {8, 16}) run<7>("entry, FHFMA split", w);
  for (int w : {8, 16}) run<8>("entry, truncation split", w);
  for (int w : {8, 16}) run<9>("F2FP pack (per entry)", w);
  for (int w : {8, 16}) run<10>("HADD2.F32 unpack (per entry)", w);
  return 0;
}

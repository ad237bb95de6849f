// Warp-level mma.sync (legacy HMMA path) throughput on sm_100a: m16n8k16
// f32 += f16 x f16, independent accumulator chains per warp. Reports TFLOP/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hmma_bench tools/hmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IT = 4096;
constexpr int CH = 8;  // independent accumulators per warp

__global__ void kern(float* out, long long* cyc) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);
  for (int i = 0; i < 2; ++i) b[i] = 0x3c003c00u ^ (threadIdx.x * 3 + i);
  float c[CH][4];
  for (int k = 0; k < CH; ++k)
    for (int i = 0; i < 4; ++i) c[k][i] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  long long t1 = clock64();
  float s = 0;
  for (int k = 0; k < CH; ++k)
    for (int i = 0; i < 4; ++i) s += c[k][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* o;
  long long* c;
  cudaMalloc(&o, 148 * 1024 * 4);
  cudaMalloc(&c, 148 * 8);
  for (int warps : {4, 8, 16}) {
    kern<<<148, 32 * warps>>>(o, c);
    cudaError_t e = cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double flop_per_sm = 2.0 * 16 * 8 * 16 * (double)IT * CH * warps;
    const double per_clk = flop_per_sm / h;
    printf("warps/SM=%2d: %.0f FLOP/clk/SM = %.0f TFLOP/s at 1965 MHz x 148 SMs %s\n", warps, per_clk,
           per_clk * 148 * 1.965e9 / 1e12, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}

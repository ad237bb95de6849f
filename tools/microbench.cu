// Pipe-throughput microbenchmarks for the K1 instruction mix on B200 (sm_100a).
// Each kernel runs a long dependent-free loop of one instruction class with
// enough independent chains per thread to saturate the pipe; throughput is
// reported as warp-instructions per SM per clock (cycles from clock64()).
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 4096

__global__ void k_ffma(float* out, float a, float b, long long* cyc) {
  float x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fmaf(x[c], a, b + c);  // 3-reg
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma(double* out, double a, double b, long long* cyc) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ex2(float* out, float a, long long* cyc) {
  float x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = -(threadIdx.x * 1e-3f + c * 0.1f);
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c])); x[c] = y; }
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_f2d(double* out, float a, long long* cyc) {
  float x[CHAINS]; double acc[CHAINS];
  for (int c = 0; c < CHAINS; ++c) { x[c] = threadIdx.x * 1e-3f + c; acc[c] = 0; }
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) { double d; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(x[c])); acc[c] = d; x[c] = __int_as_float(__double2hiint(d) ^ i); }
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename F>
void run(const char* name, F launch, int blocks, int threads, long long* dcyc, double ops_per_thread_iter) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[4096]; cudaMemcpy(h, dcyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < blocks; ++i) mean += h[i]; mean /= blocks;
  double thread_ops = (double)blocks * threads * ITERS * ops_per_thread_iter;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // per-SM per-clock thread-ops, assuming blocks spread evenly and resident together
  double per_sm_clk = thread_ops / sms / mean;
  printf("%-8s  %.3f ms  %.3e thread-op/s  cycles(mean CTA)=%.0f  => %.1f thread-ops/SM/clk  (implied clock %.0f MHz)\n",
         name, ms, thread_ops / (ms * 1e-3), mean, per_sm_clk, mean / (ms * 1e-3) / 1e6);
  cudaError_t err = cudaGetLastError(); if (err) printf("err %s\n", cudaGetErrorString(err));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz L2=%d MB smem/SM=%zu regs/SM=%d\n", p.name, sms, clk, p.l2CacheSize >> 20,
         p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor);
  int threads = 512, blocks = sms * 2;  // 32 warps/SM
  float* f; double* d; long long* cyc;
  cudaMalloc(&f, blocks * threads * 4); cudaMalloc(&d, blocks * threads * 8); cudaMalloc(&cyc, 4096 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    run("ffma", [&] { k_ffma<<<blocks, threads>>>(f, 0.999f, 1e-3f, cyc); }, blocks, threads, cyc, CHAINS);
    run("dfma", [&] { k_dfma<<<blocks, threads>>>(d, 0.999, 1e-3, cyc); }, blocks, threads, cyc, CHAINS);
    run("ex2", [&] { k_ex2<<<blocks, threads>>>(f, 0.5f, cyc); }, blocks, threads, cyc, CHAINS);
    run("f2f.f64", [&] { k_f2d<<<blocks, threads>>>(d, 0.5f, cyc); }, blocks, threads, cyc, CHAINS);
  }
  return 0;
}

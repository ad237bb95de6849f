// Thread <-> (lane, column) mapping of tcgen05.st shapes 16x64b, 16x128b,
// 16x256b (sm_100a): warp 0 stores value (1000*shape + 100*t + r) from thread
// t register r, then every lane's 8 columns are read back with 32x32b.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tmem_shape_check tools/tmem_shape_check.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void kern(unsigned* out) {
  __shared__ unsigned tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(saddr(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned tmem = tslot;
  if (warp == 0) {
    // clear columns 0..31 of lanes 0..31
    unsigned z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int c = 0; c < 32; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + c),
                   "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    // 16x64b.x1: 1 register per thread -> columns 0..1
    unsigned v1 = 1000 + 100 * lane + 0;
    asm volatile("tcgen05.st.sync.aligned.16x64b.x1.b32 [%0], {%1};" ::"r"(tmem + 0u), "r"(v1) : "memory");
    // 16x128b.x1: 2 registers -> columns 8..
    unsigned v2a = 2000 + 100 * lane + 0, v2b = 2000 + 100 * lane + 1;
    asm volatile("tcgen05.st.sync.aligned.16x128b.x1.b32 [%0], {%1,%2};" ::"r"(tmem + 8u), "r"(v2a), "r"(v2b) : "memory");
    // 16x256b.x1: 4 registers -> columns 16..
    unsigned v3[4];
    for (int r = 0; r < 4; ++r) v3[r] = 3000 + 100 * lane + r;
    asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(tmem + 16u), "r"(v3[0]),
                 "r"(v3[1]), "r"(v3[2]), "r"(v3[3]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    unsigned r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
          "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int c = 0; c < 32; ++c) out[lane * 32 + c] = r[c];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
  }
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 32 * 32 * 4);
  kern<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned h[32 * 32];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("%s\nvalue = 1000*shape(1:16x64b 2:16x128b 3:16x256b) + 100*thread + register\n", e ? cudaGetErrorString(e) : "ok");
  for (int lane = 0; lane < 32; ++lane) {
    printf("lane %2d:", lane);
    for (int c = 0; c < 24; ++c) printf(" %4u", h[lane * 32 + c]);
    printf("\n");
  }
  return 0;
}

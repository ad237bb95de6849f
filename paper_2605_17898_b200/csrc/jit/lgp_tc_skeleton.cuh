// JIT skeleton of the tensor-core fused matvec (K1-TC) for kernel trees whose
// leaves are all functions of r^2 (RBF / Matern-3/2 / Matern-5/2, with Scale,
// Sum, Product), D >= 4.
//
// Prepended by lgp_codegen.cpp: lgp_jit_abi.h, #defines LGP_D, LGP_TC_KD
// (augmented K of the distance GEMM, multiple of 8), LGP_TC_N (RHS per pass,
// 16 or 32), LGP_TC_G (chunks per FP32 accumulation group), LGP_TC_STAGES, and
// the generated lgp_tc_prep_point() / lgp_tc_k().
//
// Per CTA: 128 rows (one TMEM lane each) x one column segment, streamed in
// 64-column chunks.
//
//   GEMM1 (tcgen05.mma kind::tf32, 3xTF32 split, A and B from SMEM):
//       S'[128 x 64] = A1 . B1^T with a_i = [c_i, |c_i|^2, 1], b_j = [-2 c_j, 1, |c_j|^2]
//       so S'_ij = r^2_ij (lengthscale-scaled) lands in TMEM directly.
//   epilogue (8 warps, SIMT): r^2 -> k (the tree, one MUFU.EX2 per exp) ->
//       TF32 hi/lo split -> tcgen05.st back into TMEM as the A operand of
//   GEMM2 (kind::tf32, 3xTF32, A = P from TMEM, B = V tile from SMEM):
//       D2[128 x N] += P[128 x 64] . V[64 x N]
//   D2 (FP32, TMEM) is drained every LGP_TC_G chunks of a warpgroup into FP64
//   registers; the two epilogue warpgroups' FP64 sums are combined in a fixed
//   order and written as this segment's partial (deterministic).
//
// Warp roles: warp 0 = TMA bulk-copy producer (+ TMEM allocator), warp 1 =
// MMA issuer (one thread), warps 2..5 / 6..9 = epilogue warpgroups 0 / 1
// (even / odd chunks, each with its own TMEM buffers), so chunk c's epilogue
// overlaps chunk c+1's GEMM1 and chunk c-1's GEMM2.

#define TC_CH 64
#define TC_THREADS 320
#define TC_A1_FLOATS (128 * LGP_TC_KD)
#define TC_B1_FLOATS (TC_CH * LGP_TC_KD)
#define TC_V_FLOATS (LGP_TC_N * TC_CH)
#define TC_A1_BYTES (2 * TC_A1_FLOATS * 4)
#define TC_B1_BYTES (2 * TC_B1_FLOATS * 4)
#define TC_V_BYTES (2 * TC_V_FLOATS * 4)
#define TC_STAGE_BYTES (TC_B1_BYTES + TC_V_BYTES)
#define TC_COMB_BYTES (128 * LGP_TC_N * 8)
#define TC_NBARS (13 + 2 * LGP_TC_STAGES)
#define TC_SMEM_BYTES (TC_A1_BYTES + LGP_TC_STAGES * TC_STAGE_BYTES + TC_COMB_BYTES + TC_NBARS * 8 + 16)

// barrier slots
#define B_AFULL 0
#define B_SFULL(s) (1 + (s))
#define B_SEMPTY(s) (1 + LGP_TC_STAGES + (s))
#define B_D1FULL(w) (1 + 2 * LGP_TC_STAGES + (w))
#define B_PFULL(w) (3 + 2 * LGP_TC_STAGES + (w))
#define B_D2FULL(w, b) (5 + 2 * LGP_TC_STAGES + 2 * (w) + (b))
#define B_D2EMPTY(w, b) (9 + 2 * LGP_TC_STAGES + 2 * (w) + (b))

__device__ __forceinline__ float lgp_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float lgp_sqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ unsigned lgp_saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void lgp_mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void lgp_mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void lgp_mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void lgp_mbar_wait(unsigned bar, unsigned parity) {
  unsigned ok = 0;
#ifdef LGP_TC_WATCHDOG
  unsigned long long spins = 0;
#endif
  while (!ok) {
#ifdef LGP_TC_WATCHDOG
    if (++spins > (1ull << 28)) asm volatile("trap;");
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void lgp_bulk_g2s(unsigned dst, const void* src, unsigned bytes,
                                             unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// UMMA shared-memory descriptor: K-major, no swizzle (canonical
// ((8,m),2):((16B,SBO),LBO)), LBO = 128 B between the two 16-byte K halves,
// SBO between 8-row core-matrix groups, version 1 (sm_100).
__device__ __forceinline__ unsigned long long lgp_sdesc(unsigned saddr, unsigned sbo) {
  return (unsigned long long)((saddr >> 4) & 0x3FFFu) | ((unsigned long long)(128u >> 4) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void lgp_mma_ss(unsigned d, unsigned long long ad, unsigned long long bd,
                                           unsigned idesc, unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void lgp_mma_ts(unsigned d, unsigned a_tmem, unsigned long long bd,
                                           unsigned idesc, unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void lgp_mma_commit(unsigned bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

__device__ __forceinline__ void lgp_tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void lgp_tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

#define LGP_R8(a, o) "=r"(a[o + 0]), "=r"(a[o + 1]), "=r"(a[o + 2]), "=r"(a[o + 3]), \
                     "=r"(a[o + 4]), "=r"(a[o + 5]), "=r"(a[o + 6]), "=r"(a[o + 7])
#define LGP_W8(a, o) "r"(a[o + 0]), "r"(a[o + 1]), "r"(a[o + 2]), "r"(a[o + 3]), \
                     "r"(a[o + 4]), "r"(a[o + 5]), "r"(a[o + 6]), "r"(a[o + 7])

__device__ __forceinline__ void lgp_tmem_ld32(unsigned taddr, unsigned (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%"
      "15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : LGP_R8(v, 0), LGP_R8(v, 8), LGP_R8(v, 16), LGP_R8(v, 24)
      : "r"(taddr));
}

__device__ __forceinline__ void lgp_tmem_ld16(unsigned taddr, unsigned* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%"
      "15}, [%16];"
      : LGP_R8(v, 0), LGP_R8(v, 8)
      : "r"(taddr));
}

__device__ __forceinline__ void lgp_tmem_st32(unsigned taddr, const unsigned (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%"
      "14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      LGP_W8(v, 0), LGP_W8(v, 8), LGP_W8(v, 16), LGP_W8(v, 24)
      : "memory");
}

__device__ __forceinline__ void lgp_tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void lgp_tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// offset (floats) of element (row r, k) in a K-major no-swizzle tile with KD
// columns: 8-row core-matrix groups of (KD/4) x 128 B, K halves 128 B apart
__device__ __forceinline__ int lgp_tc_off(int r, int k, int kd) {
  return (r >> 3) * (kd * 8) + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

__device__ __forceinline__ void lgp_tf32_split(double v, float& hi, float& lo) {
  const float f = (float)v;
  hi = __uint_as_float(__float_as_uint(f) & 0xFFFFE000u);
  lo = (float)(v - (double)hi);
}

// ------------------------------------------------------------ features
// rows (tile_rows = 128, fr = A1) and columns (tile_rows = 64, fc = B1)
extern "C" __global__ void lgp_tc_prep(LgpPrepArgs p, int tile_rows, int is_col) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_pad) return;
  double f[LGP_TC_KD];
#pragma unroll
  for (int k = 0; k < LGP_TC_KD; ++k) f[k] = 0.0;
  if (i < p.n) {
    double x[LGP_D];
    const double* xp = p.x + (p.row0 + i) * LGP_D;
#pragma unroll
    for (int d = 0; d < LGP_D; ++d) x[d] = xp[d];
    lgp_tc_prep_point(x, p, is_col, f);
  }
  float* base = is_col ? p.fc : p.fr;
  const long long tile = i / tile_rows;
  const int r = (int)(i % tile_rows);
  float* hi = base + tile * 2 * tile_rows * LGP_TC_KD;
  float* lo = hi + tile_rows * LGP_TC_KD;
#pragma unroll
  for (int k4 = 0; k4 < LGP_TC_KD; k4 += 4) {
    float h[4], l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) lgp_tf32_split(f[k4 + q], h[q], l[q]);
    const int o = lgp_tc_off(r, k4, LGP_TC_KD);
    *reinterpret_cast<float4*>(hi + o) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(lo + o) = make_float4(l[0], l[1], l[2], l[3]);
  }
}

// ------------------------------------------------------------------ K1-TC
extern "C" __global__ void __launch_bounds__(TC_THREADS, 1) lgp_matvec_tc(const LgpTcArgs a) {
  if (a.done != nullptr && *a.done) return;
  const int item = blockIdx.x;
  const int rb = item % a.n_rb;
  const int rest = item / a.n_rb;
  const int seg = rest % a.n_seg;
  const int pass = rest / a.n_seg;
  const int tile0 = seg * a.tiles_per_seg;
  int nch = a.n_tiles - tile0;
  if (nch > a.tiles_per_seg) nch = a.tiles_per_seg;

  extern __shared__ __align__(1024) unsigned char tc_smem[];
  float* a1s = reinterpret_cast<float*>(tc_smem);
  unsigned char* stg = tc_smem + TC_A1_BYTES;
  double* comb = reinterpret_cast<double*>(stg + LGP_TC_STAGES * TC_STAGE_BYTES);
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(reinterpret_cast<unsigned char*>(comb) + TC_COMB_BYTES);
  unsigned* tslot = reinterpret_cast<unsigned*>(bars + TC_NBARS);
  const unsigned bar0 = lgp_saddr(bars);
#define BAR(i) (bar0 + 8u * (unsigned)(i))

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    lgp_mbar_init(BAR(B_AFULL), 1);
    for (int s = 0; s < LGP_TC_STAGES; ++s) {
      lgp_mbar_init(BAR(B_SFULL(s)), 1);
      lgp_mbar_init(BAR(B_SEMPTY(s)), 1);
    }
    for (int w = 0; w < 2; ++w) {
      lgp_mbar_init(BAR(B_D1FULL(w)), 1);
      lgp_mbar_init(BAR(B_PFULL(w)), 4);
      for (int b = 0; b < 2; ++b) {
        lgp_mbar_init(BAR(B_D2FULL(w, b)), 1);
        lgp_mbar_init(BAR(B_D2EMPTY(w, b)), 4);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     lgp_saddr(tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  lgp_tc_fence_before();
  __syncthreads();
  lgp_tc_fence_after();
  const unsigned tmem = *tslot;
  // TMEM columns: D1[w] (S' then P_hi) 64 each, L[w] (P_lo) 64 each, D2[w][b] N each
#define T_D1(w) (tmem + 64u * (unsigned)(w))
#define T_L(w) (tmem + 128u + 64u * (unsigned)(w))
#define T_D2(w, b) (tmem + 256u + (unsigned)LGP_TC_N * (2u * (unsigned)(w) + (unsigned)(b)))

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ producer (TMA bulk)
      lgp_mbar_expect_tx(BAR(B_AFULL), TC_A1_BYTES);
      lgp_bulk_g2s(lgp_saddr(a1s), a.a1 + (size_t)rb * 2 * TC_A1_FLOATS, TC_A1_BYTES, BAR(B_AFULL));
      for (int c = 0; c < nch; ++c) {
        const int s = c % LGP_TC_STAGES;
        if (c >= LGP_TC_STAGES) lgp_mbar_wait(BAR(B_SEMPTY(s)), ((c / LGP_TC_STAGES) - 1) & 1);
        const unsigned dst = lgp_saddr(stg + (size_t)s * TC_STAGE_BYTES);
        lgp_mbar_expect_tx(BAR(B_SFULL(s)), TC_STAGE_BYTES);
        lgp_bulk_g2s(dst, a.b1 + (size_t)(tile0 + c) * 2 * TC_B1_FLOATS, TC_B1_BYTES,
                     BAR(B_SFULL(s)));
        lgp_bulk_g2s(dst + TC_B1_BYTES,
                     a.v + ((size_t)pass * a.n_tiles + tile0 + c) * 2 * TC_V_FLOATS, TC_V_BYTES,
                     BAR(B_SFULL(s)));
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      const unsigned idesc1 = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(TC_CH >> 3) << 17) |
                              ((unsigned)(128 >> 4) << 24);
      const unsigned idesc2 = (1u << 4) | (2u << 7) | (2u << 10) |
                              ((unsigned)(LGP_TC_N >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
      const unsigned a_hi = lgp_saddr(a1s), a_lo = a_hi + TC_A1_FLOATS * 4;
      const unsigned sbo_k = LGP_TC_KD * 32;
      lgp_mbar_wait(BAR(B_AFULL), 0);
      for (int c = 0; c <= nch; ++c) {
        if (c < nch) {
          const int s = c % LGP_TC_STAGES;
          lgp_mbar_wait(BAR(B_SFULL(s)), (c / LGP_TC_STAGES) & 1);
          lgp_tc_fence_after();
          const unsigned b_hi = lgp_saddr(stg + (size_t)s * TC_STAGE_BYTES);
          const unsigned b_lo = b_hi + TC_B1_FLOATS * 4;
          const unsigned d = T_D1(c & 1);
#pragma unroll
          for (int kk = 0; kk < LGP_TC_KD / 8; ++kk) {
            const unsigned o = 256u * kk;
            lgp_mma_ss(d, lgp_sdesc(a_hi + o, sbo_k), lgp_sdesc(b_hi + o, sbo_k), idesc1, kk > 0);
            lgp_mma_ss(d, lgp_sdesc(a_hi + o, sbo_k), lgp_sdesc(b_lo + o, sbo_k), idesc1, 1);
            lgp_mma_ss(d, lgp_sdesc(a_lo + o, sbo_k), lgp_sdesc(b_hi + o, sbo_k), idesc1, 1);
          }
          lgp_mma_commit(BAR(B_D1FULL(c & 1)));
        }
        if (c >= 1) {
          // GEMM2 of chunk cc = c - 1
          const int cc = c - 1;
          const int w = cc & 1, k = cc >> 1, gi = k / LGP_TC_G, b = gi & 1;
          const bool first = (k % LGP_TC_G) == 0;
          const bool last = ((k % LGP_TC_G) == LGP_TC_G - 1) || (cc + 2 >= nch);
          lgp_mbar_wait(BAR(B_PFULL(w)), k & 1);
          if (first && gi >= 2) lgp_mbar_wait(BAR(B_D2EMPTY(w, b)), ((gi >> 1) - 1) & 1);
          lgp_tc_fence_after();
          const int s = cc % LGP_TC_STAGES;
          const unsigned v_hi = lgp_saddr(stg + (size_t)s * TC_STAGE_BYTES) + TC_B1_BYTES;
          const unsigned v_lo = v_hi + TC_V_FLOATS * 4;
          const unsigned d = T_D2(w, b);
#pragma unroll
          for (int kk = 0; kk < TC_CH / 8; ++kk) {
            const unsigned o = 256u * kk;
            lgp_mma_ts(d, T_D1(w) + 8u * kk, lgp_sdesc(v_hi + o, 2048u), idesc2,
                       (first && kk == 0) ? 0u : 1u);
            lgp_mma_ts(d, T_D1(w) + 8u * kk, lgp_sdesc(v_lo + o, 2048u), idesc2, 1u);
            lgp_mma_ts(d, T_L(w) + 8u * kk, lgp_sdesc(v_hi + o, 2048u), idesc2, 1u);
          }
          lgp_mma_commit(BAR(B_SEMPTY(s)));
          if (last) lgp_mma_commit(BAR(B_D2FULL(w, b)));
        }
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------- epilogue warpgroups
    const int w = (warp - 2) >> 2;
    const int q = warp & 3;                 // TMEM lane quarter of this warp
    const int row = 32 * q + lane;          // row within the 128-row tile
    const unsigned lanes = (unsigned)(32 * q) << 16;
    const int nloc = (nch - w + 1) >> 1;    // chunks of this warpgroup
    double acc[LGP_TC_N];
#pragma unroll
    for (int i = 0; i < LGP_TC_N; ++i) acc[i] = 0.0;

    auto drain = [&](int gi) {
      const int b = gi & 1;
      lgp_mbar_wait(BAR(B_D2FULL(w, b)), (gi >> 1) & 1);
      lgp_tc_fence_after();
#pragma unroll
      for (int h = 0; h < LGP_TC_N / 16; ++h) {
        unsigned v[16];
        lgp_tmem_ld16(T_D2(w, b) + lanes + 16u * h, v);
        lgp_tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[16 * h + i] += (double)__uint_as_float(v[i]);
      }
      lgp_tc_fence_before();
      __syncwarp();
      if (lane == 0) lgp_mbar_arrive(BAR(B_D2EMPTY(w, b)));
    };

    for (int k = 0; k < nloc; ++k) {
      lgp_mbar_wait(BAR(B_D1FULL(w)), k & 1);
      lgp_tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        unsigned s[32], hi[32], lo[32];
        lgp_tmem_ld32(T_D1(w) + lanes + 32u * h, s);
        lgp_tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float r2 = fmaxf(__uint_as_float(s[i]), 0.f);
          const float kv = lgp_tc_k(r2, a);
          const unsigned hb = __float_as_uint(kv) & 0xFFFFE000u;
          hi[i] = hb;
          lo[i] = __float_as_uint(kv - __uint_as_float(hb));
        }
        lgp_tmem_st32(T_D1(w) + lanes + 32u * h, hi);
        lgp_tmem_st32(T_L(w) + lanes + 32u * h, lo);
      }
      lgp_tmem_wait_st();
      lgp_tc_fence_before();
      __syncwarp();
      if (lane == 0) lgp_mbar_arrive(BAR(B_PFULL(w)));
      if (k >= 1 && ((k - 1) % LGP_TC_G) == LGP_TC_G - 1) drain((k - 1) / LGP_TC_G);
    }
    if (nloc >= 1) drain((nloc - 1) / LGP_TC_G);

    // combine the two warpgroups' FP64 sums in a fixed order
    if (w == 1) {
#pragma unroll
      for (int i = 0; i < LGP_TC_N; ++i) comb[row * LGP_TC_N + i] = acc[i];
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (w == 0) {
      double* out = a.partial +
                    (((size_t)seg * a.n_pass + pass) * a.n_rows_pad + (size_t)rb * 128 + row) *
                        LGP_TC_N;
#pragma unroll
      for (int i = 0; i < LGP_TC_N; i += 2) {
        const double x0 = acc[i] + comb[row * LGP_TC_N + i];
        const double x1 = acc[i + 1] + comb[row * LGP_TC_N + i + 1];
        reinterpret_cast<double2*>(out)[i / 2] = make_double2(x0, x1);
      }
    }
  }
  lgp_tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    lgp_tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
#undef BAR
#undef T_D1
#undef T_L
#undef T_D2
}

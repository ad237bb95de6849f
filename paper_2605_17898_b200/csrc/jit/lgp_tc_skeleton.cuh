// JIT skeleton of the tensor-core fused matvec (K1-TC) for kernel trees whose
// leaves are functions of r^2 (RBF / Matern-3/2 / Matern-5/2) or Periodic
// (angle addition on per-point features), with Scale / Sum / Product.
//
// Prepended by lgp_codegen.cpp: lgp_jit_abi.h, #defines LGP_D, LGP_TC_KD
// (K of the distance GEMM in FP16 halves: 3D + 4 rounded up to 16), LGP_TC_N
// (right-hand sides per pass: 8, 16, 32 or 64), LGP_TC_NSB (S buffers that fit
// next to the accumulators in TMEM), LGP_TC_G (chunks per FP32 accumulation
// group), LGP_TC_STAGES, LGP_TC_FW / P0 / PF (FP32 point features, Periodic
// block), and the generated lgp_tc_prep_point() / lgp_tc_k() / lgp_tc_kf().
//
// Per CTA: 128 rows (one TMEM lane each) x one column segment, streamed in
// 64-column chunks.
//
//   GEMM1 (tcgen05.mma kind::f16, A and B from SMEM, FP32 accumulate):
//       S'[128 x 64] = A1 . B1^T with the FP16 hi/lo split of the augmented
//       features laid side by side in K (3D + 4 halves, see lgp_tc_prep):
//       a_i = [c_hi | c_hi | c_lo | n_hi n_lo 1 1], b_j = [2c_hi | 2c_lo | 2c_hi | -1 -1 -m_hi -m_lo]
//       so S'_ij = 2 c_i.c_j - |c_i|^2 - |c_j|^2 = -r^2_ij (lengthscale-scaled)
//       lands in TMEM directly: ceil((3D+4)/16) MMAs per chunk (2 for D <= 9).
//   epilogue (8 warps, SIMT): r^2 -> k (the tree, one MUFU.EX2 per exp) ->
//       FP16 hi/lo split -> tcgen05.st back into TMEM as the A operand of
//   GEMM2 (kind::f16, A = P from TMEM as FP16 hi/lo, B = [V_hi ; V_lo] tile
//       from SMEM, FP16 hi/lo of a power-of-two column scaling):
//       up to 32 RHS:  D2[128 x 2N] += P_hi.[V_hi V_lo] + P_lo.[V_hi V_lo]
//                      (2 MMAs per 16 columns, hi / lo columns summed at the drain)
//       64 RHS:        D2[128 x N] += P_hi.V_hi + P_lo.V_hi + P_hi.V_lo
//                      (3 MMAs per 16 columns into one accumulator - half the
//                      TMEM columns; the lo.lo term, 2^-22 relative, dropped as
//                      in the distance GEMM; 12 instead of 8 MMAs per chunk
//                      cost 6 % at 16 RHS, hence only where TMEM needs it)
//   D2 (FP32, TMEM) is drained every LGP_TC_G chunks of a warpgroup into FP64
//   registers; the epilogue warpgroups' FP64 sums are combined in a fixed
//   order and written as this segment's partial (deterministic).
//
// Warp roles: warp 0 = TMA bulk-copy producer (+ TMEM allocator); LGP_TC_NWG
// epilogue warpgroups, chunk c -> warpgroup c % NWG and S buffer c % NSB, each
// with its own contraction issuer (one MMA-issuing thread sustains ~60-90
// cycles per MMA). Up to 32 RHS: 3 warpgroups (16 warps, 128 registers: the
// epilogue works in two 32-column halves; MUFU needs more than two warps per
// SM sub-partition to stay busy: cfg4 t = 16 2.96 vs 3.46 ms with 2), and the
// contraction issuer of chunk c also issues the distance GEMM of chunk c + NSB
// right behind it (tcgen05.mma ops of one thread execute in issue order, so
// the GEMM may overwrite P as soon as the contraction is issued). 64 RHS: 2
// warpgroups (the FP64 row sums take 128 registers) and a distance-GEMM
// issuer warp that waits for each S buffer's contraction to complete
// (PEMPTY). TMEM: LGP_TC_NSB S buffers of 64 columns (S' in FP32, then P
// packed FP16 hi | lo in place) + LGP_TC_D2B D2 accumulators per warpgroup (2N
// columns, N with 64 RHS).
//
// (Measured and dropped, round 1: CTA pairs (cta_group::2, M = 256: 5.1 vs
// 3.6 ms at cfg4 - MMA instructions are not the binding resource), distance
// tiles on mma.sync (4.2-5.3 ms), distance tiles on the FMA pipe (4.4-5.0 ms),
// 3-4 epilogue warpgroups with shared-memory row sums (4.6 ms).)

#ifndef LGP_TC_D2B
#define LGP_TC_D2B 2  // D2 accumulators per warpgroup (1: drained one chunk into the next group)
#endif
#ifndef LGP_TC_DLAG
#define LGP_TC_DLAG (LGP_TC_D2B == 1 ? 1 : (LGP_TC_G + 1) / 2)
#endif
#if LGP_TC_DLAG < 1 || LGP_TC_DLAG > LGP_TC_G
#error "LGP_TC_DLAG must be in [1, LGP_TC_G]"
#endif
// S' = -r^2 may come out a rounding error above 0; leaves that take sqrt(r^2)
// need it clamped (LGP_TC_CLAMP defined by the code generator), exp2 does not
#ifndef LGP_TC_CLAMP
#define LGP_TC_CLAMP(x) (x)
#endif

#define TC_CH 64
#ifndef LGP_TC_NWG
#define LGP_TC_NWG 2  // epilogue warpgroups (chunk c -> warpgroup c % NWG)
#endif
// distance GEMMs issued by a warp of their own (else by the contraction
// issuers, right behind the contraction that frees their S buffer)
#ifndef LGP_TC_DISTW
#define LGP_TC_DISTW (LGP_TC_NWG == 2)
#endif
// warps: producer, [distance-GEMM issuer], then per warpgroup one contraction
// issuer and four epilogue warps (3 warpgroups: 16 warps, 128 registers)
// contraction issuers: issuer i takes the chunks c = i (mod NCI)
#ifndef LGP_TC_NCI
#define LGP_TC_NCI LGP_TC_NWG
#endif
#define TC_THREADS (32 * (1 + LGP_TC_DISTW + LGP_TC_NCI + 4 * LGP_TC_NWG))
#if !LGP_TC_DISTW && LGP_TC_NSB > LGP_TC_STAGES
#error "distance GEMMs queued behind the contractions need NSB <= STAGES (ring deadlock)"
#endif
#define TC_W_CI (1 + LGP_TC_DISTW)                 // first contraction issuer
#define TC_W_EPI (1 + LGP_TC_DISTW + LGP_TC_NCI)   // first epilogue warp
#if LGP_TC_N != 8 && LGP_TC_N != 16 && LGP_TC_N != 32 && LGP_TC_N != 64
#error "K1-TC takes 8, 16, 32 or 64 right-hand sides per pass"
#endif
#define TC_KSTACK (LGP_TC_N == 64)                 // cross terms stacked in K (see above)
#define TC_N2 (TC_KSTACK ? LGP_TC_N : 2 * LGP_TC_N)  // GEMM2 N = D2 columns
// epilogue round trips per chunk: 64 RHS -> two 32-column halves
#define TC_HALVES ((LGP_TC_N == 64 || LGP_TC_NWG > 2) ? 2 : 1)
// TMEM column (within an S buffer) of the FP16x2 hi / lo words of the
// contraction's K step kk (16 chunk columns)
#define TC_PHI(kk) (TC_HALVES == 1 ? 8u * (kk) : 32u * ((kk) >> 1) + 8u * ((kk) & 1))
#define TC_PLO(kk) (TC_PHI(kk) + (TC_HALVES == 1 ? 32u : 16u))
#define TC_V_HALFS (LGP_TC_N * TC_CH)
// row / column operand tiles (FP16, UMMA K-major canonical layout)
#define TC_A1_BYTES (128 * LGP_TC_KD * 2)
#define TC_B1_BYTES (TC_CH * LGP_TC_KD * 2)
#define TC_V_BYTES (2 * TC_V_HALFS * 2)
#ifndef LGP_TC_PF
#define LGP_TC_PF 0  // Periodic (cos, sin) features per point, from offset LGP_TC_P0
#define LGP_TC_P0 0
#endif
// FP32 column features of a chunk (trees with Periodic leaves)
#define TC_C32_BYTES (LGP_TC_PF ? TC_CH * LGP_TC_FW * 4 : 0)
#define TC_STAGE_BYTES (TC_B1_BYTES + TC_V_BYTES + TC_C32_BYTES)
#define TC_COMB_BYTES ((LGP_TC_NWG - 1) * 128 * LGP_TC_N * 8)
#ifndef LGP_TC_NSB
#define LGP_TC_NSB 6   // S buffers in TMEM (64 columns each): chunk c -> buffer c % NSB
#endif
#if 64 * LGP_TC_NSB + LGP_TC_D2B * LGP_TC_NWG * TC_N2 > 512
#error "TMEM budget: S buffers + D2 accumulators exceed 512 columns"
#endif
#define TC_NBARS (1 + 2 * LGP_TC_STAGES + 3 * LGP_TC_NSB + 4 * LGP_TC_NWG)

// barrier slots
#define B_AFULL 0
#define B_SFULL(s) (1 + (s))
#define B_SEMPTY(s) (1 + LGP_TC_STAGES + (s))
#define B_S1FULL(q) (1 + 2 * LGP_TC_STAGES + (q))
#define B_PFULL(q) (1 + 2 * LGP_TC_STAGES + LGP_TC_NSB + (q))
#define B_PEMPTY(q) (1 + 2 * LGP_TC_STAGES + 2 * LGP_TC_NSB + (q))
#define B_D2FULL(w, b) (1 + 2 * LGP_TC_STAGES + 3 * LGP_TC_NSB + 2 * (w) + (b))
#define B_D2EMPTY(w, b) (1 + 2 * LGP_TC_STAGES + 3 * LGP_TC_NSB + 2 * LGP_TC_NWG + 2 * (w) + (b))

// blocking mbarrier waits let the hardware suspend the waiting thread (up to
// this many ns per try) instead of spinning: spinning producer / issuer /
// epilogue warps steal issue slots from the working warps of their SM
// sub-partition
#ifndef LGP_TC_SUSPEND_NS
#define LGP_TC_SUSPEND_NS 20000
#endif

__device__ __forceinline__ float lgp_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x (x <= 0) on the FMA pipe: x = n + f, f in [-1/2, 1/2] by the
// 1.5 * 2^23 rounding trick, degree-5 fit of 2^f (max relative error 2.3e-7 in
// FP32 Horner form, same order as MUFU.EX2), n added into the exponent field
__device__ __forceinline__ float lgp_ex2_fma(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = 1.32764783e-3f;
  p = fmaf(p, f, 9.67554189e-3f);
  p = fmaf(p, f, 5.55071309e-2f);
  p = fmaf(p, f, 2.40221202e-1f);
  p = fmaf(p, f, 6.93146944e-1f);
  p = fmaf(p, f, 1.00000012f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ float lgp_ex2x(float x, int px) {
  return px ? lgp_ex2_fma(x) : lgp_ex2(x);
}

// entries per 16 whose exp2 runs on the FMA pipe instead of MUFU (set by the
// code generator per tree)
#ifndef LGP_TC_POLY
#define LGP_TC_POLY 2
#endif

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

__device__ __forceinline__ bool lgp_mbar_test(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void lgp_mbar_wait(unsigned bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(LGP_TC_SUSPEND_NS)
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
// ((8,m),2):((16B,SBO),LBO)), LBO = 128 B between the two 16-byte K chunks of
// one instruction, SBO between 8-row core-matrix groups, version 1 (sm_100).
__device__ __forceinline__ unsigned long long lgp_sdesc(unsigned saddr, unsigned sbo) {
  return (unsigned long long)((saddr >> 4) & 0x3FFFu) | ((unsigned long long)(128u >> 4) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void lgp_mma_f16_ss(unsigned d, unsigned long long ad,
                                               unsigned long long bd, unsigned idesc,
                                               unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void lgp_mma_f16_ts(unsigned d, unsigned a_tmem, unsigned long long bd,
                                               unsigned idesc, unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
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

// 32 columns into v[0..31] / from v[0], v[2], ..., v[62] (stride-2 registers)
__device__ __forceinline__ void lgp_tmem_ld32p(unsigned taddr, unsigned* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%"
      "15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : LGP_R8(v, 0), LGP_R8(v, 8), LGP_R8(v, 16), LGP_R8(v, 24)
      : "r"(taddr));
}

#define LGP_W8S2(a, o) "r"(a[o + 0]), "r"(a[o + 2]), "r"(a[o + 4]), "r"(a[o + 6]), \
                       "r"(a[o + 8]), "r"(a[o + 10]), "r"(a[o + 12]), "r"(a[o + 14])
__device__ __forceinline__ void lgp_tmem_st32s2(unsigned taddr, const unsigned* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%"
      "14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      LGP_W8S2(v, 0), LGP_W8S2(v, 16), LGP_W8S2(v, 32), LGP_W8S2(v, 48)
      : "memory");
}

#define LGP_W4S2(a, o) "r"(a[o + 0]), "r"(a[o + 2]), "r"(a[o + 4]), "r"(a[o + 6])
// 16 columns from v[0], v[2], ..., v[30]
__device__ __forceinline__ void lgp_tmem_st16s2(unsigned taddr, const unsigned* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16};" ::"r"(taddr),
      LGP_W4S2(v, 0), LGP_W4S2(v, 8), LGP_W4S2(v, 16), LGP_W4S2(v, 24)
      : "memory");
}

__device__ __forceinline__ void lgp_tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void lgp_tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void lgp_tmem_ld8(unsigned taddr, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : LGP_R8(v, 0)
               : "r"(taddr));
}

// FP16 hi/lo split of two FP32 values, packed {lo half = x0, hi half = x1}:
// hi = RN(x), lo = RN(x - hi) with x - hi formed exactly by the mixed-precision
// FMA (FHFMA: FP16 operand, FP32 addend), no FP16 -> FP32 unpack needed
__device__ __forceinline__ void lgp_split_f16x2(float x0, float x1, unsigned& hi, unsigned& lo) {
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

// offset (halves) of element (row r, k) in a K-major no-swizzle FP16 tile with
// KH columns: 8-row core-matrix groups of (KH/8) x 128 B, K chunks 128 B apart
__device__ __forceinline__ int lgp_tc_off(int r, int k, int kh) {
  return (r >> 3) * (kh * 8) + (k >> 3) * 64 + (r & 7) * 8 + (k & 7);
}

// FP16 hi/lo split of an FP64 value (round to nearest both times)
__device__ __forceinline__ void lgp_f16_split(double v, unsigned short& hi, unsigned short& lo) {
  unsigned short h, l;
  double hd;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(v));
  asm("cvt.f64.f16 %0, %1;" : "=d"(hd) : "h"(h));
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(l) : "d"(v - hd));
  hi = h;
  lo = l;
}

// ------------------------------------------------------------ features
// rows (tile_rows = 128, fr = A1) and columns (tile_rows = 64, fc = B1): the
// FP16 hi/lo augmented features, side by side in K (see the header comment).
// c = lengthscale-scaled centred coordinates; |c| stays far inside the FP16
// range because wide point sets are routed to the direct-distance kernel
// (MatvecOp::prepare), and tiny |c| only lose absolute precision below 2^-24.
extern "C" __global__ void lgp_tc_prep(LgpPrepArgs p, int tile_rows, int is_col) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_pad) return;
  unsigned short h[LGP_TC_KD];
#pragma unroll
  for (int k = 0; k < LGP_TC_KD; ++k) h[k] = 0;
  if (i < p.n) {
    double x[LGP_D], c[LGP_D], nn;
    const double* xp = p.x + (p.row0 + i) * LGP_D;
#pragma unroll
    for (int d = 0; d < LGP_D; ++d) x[d] = xp[d];
    lgp_tc_prep_point(x, p, c, &nn);
    unsigned short nh, nl;
    lgp_f16_split(nn, nh, nl);
#pragma unroll
    for (int d = 0; d < LGP_D; ++d) {
      unsigned short ch, cl;
      lgp_f16_split(is_col ? 2.0 * c[d] : c[d], ch, cl);
      h[d] = ch;
      h[LGP_D + d] = is_col ? cl : ch;
      h[2 * LGP_D + d] = is_col ? ch : cl;
    }
    const unsigned short one = 0x3C00u, sign = 0x8000u;
    h[3 * LGP_D + 0] = is_col ? (unsigned short)(one | sign) : nh;
    h[3 * LGP_D + 1] = is_col ? (unsigned short)(one | sign) : nl;
    h[3 * LGP_D + 2] = is_col ? (unsigned short)(nh ^ sign) : one;
    h[3 * LGP_D + 3] = is_col ? (unsigned short)(nl ^ sign) : one;
    // FP32 point features [FW]: (c or 2c, -|c|^2, 0 ..), then from P0 the
    // Periodic (cos, sin) blocks (read by the epilogues of Periodic trees)
    if (p.f32 != nullptr) {
      float* f = p.f32 + i * LGP_TC_FW;
#pragma unroll
      for (int d = 0; d < LGP_D; ++d) f[d] = (float)(is_col ? 2.0 * c[d] : c[d]);
      f[LGP_D] = (float)(-nn);
#pragma unroll
      for (int k = LGP_D + 1; k < LGP_TC_FW; ++k) f[k] = 0.f;
#if LGP_TC_PF
      lgp_tc_prep_feat(x, p, f + LGP_TC_P0);
#endif
    }
  } else if (p.f32 != nullptr) {
#pragma unroll
    for (int k = 0; k < LGP_TC_FW; ++k) p.f32[i * LGP_TC_FW + k] = 0.f;
  }
  unsigned short* base = reinterpret_cast<unsigned short*>(is_col ? p.fc : p.fr) +
                         (i / tile_rows) * (long long)tile_rows * LGP_TC_KD;
  const int r = (int)(i % tile_rows);
#pragma unroll
  for (int k8 = 0; k8 < LGP_TC_KD; k8 += 8) {
    uint4 q;
    q.x = (unsigned)h[k8 + 0] | ((unsigned)h[k8 + 1] << 16);
    q.y = (unsigned)h[k8 + 2] | ((unsigned)h[k8 + 3] << 16);
    q.z = (unsigned)h[k8 + 4] | ((unsigned)h[k8 + 5] << 16);
    q.w = (unsigned)h[k8 + 6] | ((unsigned)h[k8 + 7] << 16);
    *reinterpret_cast<uint4*>(base + lgp_tc_off(r, k8, LGP_TC_KD)) = q;
  }
}

// ------------------------------------------------------------------ K1-TC
extern "C" __global__ void __launch_bounds__(TC_THREADS, 1) lgp_matvec_tc(const LgpTcArgs a) {
  if (a.done != nullptr && *a.done) return;
  const int rb = blockIdx.x % a.n_rb;
  const int rest = blockIdx.x / a.n_rb;
  const int seg = a.seg_base + rest % a.n_seg;  // n_seg: the segments of this launch
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
    for (int q = 0; q < LGP_TC_NSB; ++q) {
      lgp_mbar_init(BAR(B_S1FULL(q)), 1);
      lgp_mbar_init(BAR(B_PFULL(q)), 4);
      lgp_mbar_init(BAR(B_PEMPTY(q)), 1);
    }
    for (int w = 0; w < LGP_TC_NWG; ++w)
      for (int b = 0; b < 2; ++b) {
        lgp_mbar_init(BAR(B_D2FULL(w, b)), 1);
        lgp_mbar_init(BAR(B_D2EMPTY(w, b)), 4);
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
  // TMEM columns: S buffer q: 64 FP32 columns of S', then P packed FP16 (hi in
  // columns 0..31, lo in 32..63); D2[w][b]: 2N columns (P.V_hi | P.V_lo)
#define T_SB(q) (tmem + 64u * (unsigned)(q))
#define T_D2(w, b) \
  (tmem + 64u * LGP_TC_NSB + (unsigned)TC_N2 * ((unsigned)LGP_TC_D2B * (unsigned)(w) + (unsigned)(b)))

  // instruction descriptors: FP32 accumulate, FP16 A and B, K-major, M = 128.
  // Shared-memory descriptors are precomputed: the start-address field is
  // linear (a K step of 256 B adds 16, a stage adds STAGE_BYTES/16).
  const unsigned idesc1 = (1u << 4) | ((unsigned)(TC_CH >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
  const unsigned idesc2 = (1u << 4) | ((unsigned)(TC_N2 >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
  const unsigned long long dk = lgp_sdesc(0u, LGP_TC_KD * 16);
  const unsigned long long dv = lgp_sdesc(0u, 1024u);
  const unsigned stg0 = lgp_saddr(stg) >> 4;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ producer (TMA bulk)
      lgp_mbar_expect_tx(BAR(B_AFULL), TC_A1_BYTES);
      lgp_bulk_g2s(lgp_saddr(a1s), a.a1 + (size_t)rb * (TC_A1_BYTES / 4), TC_A1_BYTES, BAR(B_AFULL));
      const unsigned char* vbase = reinterpret_cast<const unsigned char*>(a.v);
      for (int c = 0; c < nch; ++c) {
        const int s = c % LGP_TC_STAGES;
        if (c >= LGP_TC_STAGES) lgp_mbar_wait(BAR(B_SEMPTY(s)), ((c / LGP_TC_STAGES) - 1) & 1);
        const unsigned dst = lgp_saddr(stg + (size_t)s * TC_STAGE_BYTES);
        lgp_mbar_expect_tx(BAR(B_SFULL(s)), TC_STAGE_BYTES);
        lgp_bulk_g2s(dst, reinterpret_cast<const unsigned char*>(a.b1) + (size_t)(tile0 + c) * TC_B1_BYTES,
                     TC_B1_BYTES, BAR(B_SFULL(s)));
        lgp_bulk_g2s(dst + TC_B1_BYTES, vbase + ((size_t)pass * a.n_tiles + tile0 + c) * TC_V_BYTES,
                     TC_V_BYTES, BAR(B_SFULL(s)));
#if LGP_TC_PF
        lgp_bulk_g2s(dst + TC_B1_BYTES + TC_V_BYTES,
                     reinterpret_cast<const unsigned char*>(a.c32) + (size_t)(tile0 + c) * TC_C32_BYTES,
                     TC_C32_BYTES, BAR(B_SFULL(s)));
#endif
      }
    }
    __syncwarp();
#if LGP_TC_DISTW
  } else if (warp == 1) {
    if (lane == 0) {
      // --------------------------------------------- distance-GEMM issuer
      // every chunk in order, once it is staged and its S buffer's previous
      // contraction has completed (PEMPTY)
      const unsigned long long a_d = dk + (lgp_saddr(a1s) >> 4);
      lgp_mbar_wait(BAR(B_AFULL), 0);
      for (int c = 0; c < nch; ++c) {
        const int q = c % LGP_TC_NSB;
        const int s = c % LGP_TC_STAGES;
        lgp_mbar_wait(BAR(B_SFULL(s)), (c / LGP_TC_STAGES) & 1);
        if (c >= LGP_TC_NSB) lgp_mbar_wait(BAR(B_PEMPTY(q)), ((c / LGP_TC_NSB) - 1) & 1);
        lgp_tc_fence_after();
        const unsigned long long b_d = dk + stg0 + (unsigned)s * (TC_STAGE_BYTES >> 4);
#pragma unroll
        for (int kk = 0; kk < LGP_TC_KD / 16; ++kk)
          lgp_mma_f16_ss(T_SB(q), a_d + 16u * kk, b_d + 16u * kk, idesc1, kk > 0);
        lgp_mma_commit(BAR(B_S1FULL(q)));
      }
    }
    __syncwarp();
#endif
  } else if (warp < TC_W_EPI) {
    if (lane == 0) {
      // -------------------------------------------- contraction issuers
      // each epilogue warpgroup w has its own contraction issuer that owns its
      // D2 accumulators
      const int ci = warp - TC_W_CI;
      const unsigned long long a_d = dk + (lgp_saddr(a1s) >> 4);
      // distance GEMM of chunk c into S buffer c % NSB, once its stage is in
      auto dist = [&](int c) {
        const int q = c % LGP_TC_NSB, s = c % LGP_TC_STAGES;
        lgp_mbar_wait(BAR(B_SFULL(s)), (c / LGP_TC_STAGES) & 1);
        lgp_tc_fence_after();
        const unsigned long long b_d = dk + stg0 + (unsigned)s * (TC_STAGE_BYTES >> 4);
#pragma unroll
        for (int kk = 0; kk < LGP_TC_KD / 16; ++kk)
          lgp_mma_f16_ss(T_SB(q), a_d + 16u * kk, b_d + 16u * kk, idesc1, kk > 0);
        lgp_mma_commit(BAR(B_S1FULL(q)));
      };
      if (!LGP_TC_DISTW) {
        lgp_mbar_wait(BAR(B_AFULL), 0);
        for (int c = ci; c < LGP_TC_NSB && c < nch; c += LGP_TC_NCI) dist(c);
      }
      for (int c = ci; c < nch; c += LGP_TC_NCI) {
        // chunk c: warpgroup w, its k-th chunk (of nloc)
        const int w = c % LGP_TC_NWG, k = c / LGP_TC_NWG;
        const int nloc = (nch - w + LGP_TC_NWG - 1) / LGP_TC_NWG;
        const int q = c % LGP_TC_NSB;
        const int gi = k / LGP_TC_G, b = gi % LGP_TC_D2B;
        const bool first = (k % LGP_TC_G) == 0;
        const bool last = ((k % LGP_TC_G) == LGP_TC_G - 1) || (k == nloc - 1);
        lgp_mbar_wait(BAR(B_PFULL(q)), (c / LGP_TC_NSB) & 1);
        if (first && gi >= LGP_TC_D2B) lgp_mbar_wait(BAR(B_D2EMPTY(w, b)), ((gi / LGP_TC_D2B) - 1) & 1);
        lgp_tc_fence_after();
        const int s = c % LGP_TC_STAGES;
        // B = V_hi (rows 0..N-1 of the staged V tile) and V_lo (rows N..2N-1)
        const unsigned long long v_d = dv + stg0 + (unsigned)s * (TC_STAGE_BYTES >> 4) + (TC_B1_BYTES >> 4);
        const unsigned d = T_D2(w, b);
        const unsigned p = T_SB(q);
#pragma unroll
        for (int kk = 0; kk < TC_CH / 16; ++kk) {
          const unsigned o = 16u * kk;
          lgp_mma_f16_ts(d, p + TC_PHI(kk), v_d + o, idesc2, (first && kk == 0) ? 0u : 1u);
          lgp_mma_f16_ts(d, p + TC_PLO(kk), v_d + o, idesc2, 1u);
#if TC_KSTACK
          lgp_mma_f16_ts(d, p + TC_PHI(kk), v_d + ((unsigned)(LGP_TC_N * 128) >> 4) + o, idesc2, 1u);
#endif
        }
        lgp_mma_commit(BAR(B_SEMPTY(s)));
        if (last) lgp_mma_commit(BAR(B_D2FULL(w, b)));
        // the next chunk on this S buffer: tcgen05.mma ops of one thread run
        // in issue order, so its distance GEMM may overwrite P right behind
        // this contraction (no wait for the contraction's completion)
#if LGP_TC_DISTW
        lgp_mma_commit(BAR(B_PEMPTY(q)));
#else
        if (c + LGP_TC_NSB < nch) dist(c + LGP_TC_NSB);
#endif
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------- epilogue warpgroups
    const int w = (warp - TC_W_EPI) >> 2;
    const int q4 = warp & 3;                // TMEM lane quarter of this warp
    const int row = 32 * q4 + lane;         // row within the 128-row tile
    const unsigned lanes = (unsigned)(32 * q4) << 16;
    const int nloc = nch > w ? (nch - w + LGP_TC_NWG - 1) / LGP_TC_NWG : 0;  // chunks of this warpgroup
    double acc[LGP_TC_N];
#pragma unroll
    for (int i = 0; i < LGP_TC_N; ++i) acc[i] = 0.0;
#if LGP_TC_PF
    float frp[LGP_TC_PF];  // this thread's row: Periodic (cos, sin) features
#pragma unroll
    for (int f = 0; f < LGP_TC_PF; ++f)
      frp[f] = a.r32[((size_t)rb * 128 + row) * LGP_TC_FW + LGP_TC_P0 + f];
#endif

    auto drain = [&](int gi) {
      const int b = gi % LGP_TC_D2B;
      lgp_mbar_wait(BAR(B_D2FULL(w, b)), (gi / LGP_TC_D2B) & 1);
      lgp_tc_fence_after();
      // column i: RHS i of the pass (up to 32 RHS: P.V_hi in columns
      // 0..N-1, P.V_lo in N..2N-1, both added)
#pragma unroll
      for (int h = 0; h < (TC_KSTACK ? 1 : 2); ++h) {
#if LGP_TC_N == 8
        unsigned v[8];
        lgp_tmem_ld8(T_D2(w, b) + lanes + 8u * h, v);
        lgp_tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += (double)__uint_as_float(v[i]);
#else
#pragma unroll
        for (int b16 = 0; b16 < LGP_TC_N / 16; ++b16) {
          unsigned v[16];
          lgp_tmem_ld16(T_D2(w, b) + lanes + (unsigned)(LGP_TC_N * h + 16 * b16), v);
          lgp_tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[16 * b16 + i] += (double)__uint_as_float(v[i]);
        }
#endif
      }
      lgp_tc_fence_before();
      __syncwarp();
      if (lane == 0) lgp_mbar_arrive(BAR(B_D2EMPTY(w, b)));
    };

    for (int k = 0; k < nloc; ++k) {
      const int c = LGP_TC_NWG * k + w;
      const int q = c % LGP_TC_NSB;
      const unsigned sb = T_SB(q) + lanes;
      lgp_mbar_wait(BAR(B_S1FULL(q)), (c / LGP_TC_NSB) & 1);
      lgp_tc_fence_after();
#if LGP_TC_PF
      // column Periodic features of this chunk, staged with its B tile (the
      // stage is released only after this chunk's contraction)
      const int cpf = c;
      lgp_mbar_wait(BAR(B_SFULL(cpf % LGP_TC_STAGES)), (cpf / LGP_TC_STAGES) & 1);
      const float* cfp = reinterpret_cast<const float*>(stg + (size_t)(cpf % LGP_TC_STAGES) * TC_STAGE_BYTES +
                                                        TC_B1_BYTES + TC_V_BYTES) + LGP_TC_P0;
#define TC_KJ(x, pxv, j) lgp_tc_kf((x), a, (pxv), frp, cfp + (j) * LGP_TC_FW)
#else
#define TC_KJ(x, pxv, j) lgp_tc_k((x), a, (pxv))
#endif
#if TC_HALVES == 1
      // all 64 columns in one round trip; P overwrites S' in the same
      // registers: s[2m] = FP16x2 hi of entries (2m, 2m+1), s[2m+1] = lo
      unsigned s[64];
      lgp_tmem_ld32p(sb, s);
      lgp_tmem_ld32p(sb + 32u, s + 32);
      lgp_tmem_wait_ld();
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const int px = (m & 7) < (LGP_TC_POLY + 1) / 2 ? 1 : 0;
        const int px1 = (m & 7) < LGP_TC_POLY / 2 ? 1 : 0;
        const float k0 = TC_KJ(LGP_TC_CLAMP(__uint_as_float(s[2 * m])), px, 2 * m);
        const float k1 = TC_KJ(LGP_TC_CLAMP(__uint_as_float(s[2 * m + 1])), px1, 2 * m + 1);
        lgp_split_f16x2(k0, k1, s[2 * m], s[2 * m + 1]);
      }
      lgp_tmem_st32s2(sb, s);            // hi pairs -> columns 0..31
      lgp_tmem_st32s2(sb + 32u, s + 1);  // lo pairs -> columns 32..63
#else
      // two 32-column halves (registers: the FP64 row sums of 64 RHS take
      // 128); half h's P words stay inside its own columns: hi -> 32h + 0..15,
      // lo -> 32h + 16..31 (the next half's S' columns are not touched)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        unsigned s[32];
        lgp_tmem_ld32p(sb + 32u * h, s);
        lgp_tmem_wait_ld();
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const int px = (m & 7) < (LGP_TC_POLY + 1) / 2 ? 1 : 0;
          const int px1 = (m & 7) < LGP_TC_POLY / 2 ? 1 : 0;
          const float k0 = TC_KJ(LGP_TC_CLAMP(__uint_as_float(s[2 * m])), px, 32 * h + 2 * m);
          const float k1 = TC_KJ(LGP_TC_CLAMP(__uint_as_float(s[2 * m + 1])), px1, 32 * h + 2 * m + 1);
          lgp_split_f16x2(k0, k1, s[2 * m], s[2 * m + 1]);
        }
        lgp_tmem_st16s2(sb + 32u * h, s);             // hi pairs -> columns 32h + 0..15
        lgp_tmem_st16s2(sb + 32u * h + 16u, s + 1);   // lo pairs -> columns 32h + 16..31
      }
#endif
#undef TC_KJ
      lgp_tmem_wait_st();
      lgp_tc_fence_before();
      __syncwarp();
      if (lane == 0) lgp_mbar_arrive(BAR(B_PFULL(q)));
      // drain a finished accumulation group DLAG chunks into the next one, so
      // its last contraction has long completed (DLAG <= G keeps at most two
      // groups, i.e. both D2 buffers, outstanding)
      if (k >= LGP_TC_DLAG && ((k - LGP_TC_DLAG) % LGP_TC_G) == LGP_TC_G - 1)
        drain((k - LGP_TC_DLAG) / LGP_TC_G);
    }
    for (int gi = nloc >= LGP_TC_DLAG ? (nloc - LGP_TC_DLAG) / LGP_TC_G : 0;
         gi < (nloc + LGP_TC_G - 1) / LGP_TC_G; ++gi)
      drain(gi);

    // combine the warpgroups' FP64 sums in a fixed order, undo the V scaling
    if (w > 0) {
#pragma unroll
      for (int i = 0; i < LGP_TC_N; ++i) comb[((w - 1) * LGP_TC_N + i) * 128 + row] = acc[i];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(128 * LGP_TC_NWG) : "memory");
    if (w == 0) {
#pragma unroll
      for (int u = 1; u < LGP_TC_NWG - 1; ++u)
#pragma unroll
        for (int i = 0; i < LGP_TC_N; ++i) acc[i] += comb[((u - 1) * LGP_TC_N + i) * 128 + row];
      double* out = a.partial +
                    (((size_t)seg * a.n_pass + pass) * a.n_rows_pad + (size_t)rb * 128 + row) *
                        LGP_TC_N;
      // V's power-of-two column scales are per part (column segments below /
      // from seg_split): the staged upload packs each part as it lands
      const float* sc = a.vscale + ((size_t)(seg >= a.seg_split ? 1 : 0) * a.n_pass + pass) * LGP_TC_N;
#pragma unroll
      for (int i = 0; i < LGP_TC_N; i += 2) {
        const double x0 = (acc[i] + comb[((LGP_TC_NWG - 2) * LGP_TC_N + i) * 128 + row]) * (double)sc[i];
        const double x1 = (acc[i + 1] + comb[((LGP_TC_NWG - 2) * LGP_TC_N + i + 1) * 128 + row]) * (double)sc[i + 1];
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
#undef T_SB
#undef T_D2
}

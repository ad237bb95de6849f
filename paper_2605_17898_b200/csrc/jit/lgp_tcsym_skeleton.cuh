// JIT skeleton of the symmetric tensor-core matvec (K1-TC-sym) for the square
// operator with one right-hand side: the CG matvec (K(X,X) + noise I) p.
// Appended after lgp_tc_skeleton.cuh (shares its helpers, the feature tiles
// and the generated lgp_tc_k()).
//
// Exact symmetry is what CG needs (profiles/r01_cg_tc_experiment.txt: a
// rounding-level asymmetric operator or a rounded direction vector costs 8-50 %
// more iterations), so:
//   * each unordered pair {i, j} is evaluated ONCE, in the tile of row block
//     I = block(min) and column chunk c = chunk(max), by the distance GEMM
//     (tcgen05 kind::f16, -r^2 in TMEM) and the tree on one epilogue thread,
//     and that single FP32 value k_ij feeds both out_i and out_j;
//   * the contraction stays FP64 with the exact FP64 p: the row side is one
//     DFMA per entry in the row's thread, the column side k_ij * p_i is reduced
//     over the warp's 32 rows by a transpose-reduce butterfly (after 5 levels
//     lane l holds column l) and over the 4 warps in a fixed order.
// Diagonal tiles: entries j > i go to both sides, j == i to the row side only,
// j < i are skipped (they are the pair's other orientation). Partials (row:
// per (I, segment); column: per (I, chunk)) are summed in a fixed order by
// k_tcsym_epilogue (deterministic).
//
// CTA = one row block I (128 rows, one TMEM lane each) x a segment of its
// column chunks [c0, c1) (c0 >= 2I). Warps: 0 producer (cp.async.bulk ring of
// column-feature tiles + p chunks), 1 distance-GEMM issuer, 2..9 two epilogue
// warpgroups taking even / odd chunks.

#ifndef LGP_TS_NWG
#define LGP_TS_NWG 4  // epilogue warpgroups (chunks round-robin): latency hiding
#endif
#ifndef LGP_TS_LAYOUT
#define LGP_TS_LAYOUT 1  // 1: 16x256b TMEM tiles (4 rows x 8 columns per thread); 0: 32x32b rows
#endif
#ifndef LGP_TS_PF
#define LGP_TS_PF 0  // 1: issue the second 32-column half's TMEM loads before the first half's math
#endif
#ifndef LGP_TS_ABLATE
#define LGP_TS_ABLATE 0
#endif
#ifndef LGP_TS_RFG
#define LGP_TS_RFG 0  // 1: Periodic row features through L1 (more spills: 708 vs 248 B)
#endif
#ifndef LGP_TS_POLY
#define LGP_TS_POLY 0  // entries per 16 whose exp2 runs on the FMA pipe (layout 1)
#endif
#ifndef LGP_TS_XPOSE
#define LGP_TS_XPOSE 0  // 1: column reduction through a swizzled shared-memory transpose (slower: 2.39 vs 2.30 ms); 0: butterfly
#endif
#if LGP_TS_XPOSE && LGP_TS_LAYOUT == 1
#define TS_XPOSE_DOUBLES (LGP_TS_NWG * 4 * 32 * 8)
#else
#define TS_XPOSE_DOUBLES 0
#endif
#define TS_THREADS (64 + 128 * LGP_TS_NWG)
#ifndef LGP_TS_NSB
#define LGP_TS_NSB (LGP_TS_NWG == 4 ? 8 : 6)  // S buffers of 64 TMEM columns
#endif
#define TS_NSBW (LGP_TS_NSB / LGP_TS_NWG)    // S buffers per warpgroup
#define TS_VCH_BYTES (TC_CH * 8)                        // p chunk, FP64
#define TS_F32_BYTES (LGP_TC_PF ? TC_CH * LGP_TC_FW * 4 : 0)  // column Periodic features
#define TS_STAGE_BYTES (TC_B1_BYTES + TS_VCH_BYTES + TS_F32_BYTES)
#if LGP_TC_PF && LGP_TS_LAYOUT != 1
#error "Periodic features need the 16x256b epilogue layout"
#endif
#define TS_CBUF_BYTES (LGP_TS_NWG * 2 * 4 * TC_CH * 8)  // [wg][parity][warp][64] FP64
#define TS_NBARS (1 + 2 * LGP_TC_STAGES + 2 * LGP_TS_NSB)
#define TSB_AFULL 0
#define TSB_SFULL(s) (1 + (s))
#define TSB_SEMPTY(s) (1 + LGP_TC_STAGES + (s))
#define TSB_S1FULL(q) (1 + 2 * LGP_TC_STAGES + (q))
#define TSB_SFREE(q) (1 + 2 * LGP_TC_STAGES + LGP_TS_NSB + (q))

// FP32 -> FP64 for finite non-negative kernel values without the conversion
// pipe: exponent re-bias + mantissa shift (0 maps to 2^-127, negligible)
#ifndef LGP_TS_WIDEN
#define LGP_TS_WIDEN 0  // 1: F2F.F64.F32 conversion instead of the integer re-bias
#endif
__device__ __forceinline__ double lgp_widen_nn(float f) {
#if LGP_TS_WIDEN
  return (double)f;
#else
  const unsigned b = __float_as_uint(f);
  return __hiloint2double((b >> 3) + 0x38000000u, b << 29);
#endif
}

// 16 TMEM lanes x 32 columns: thread t gets, for each 8-column block b,
// regs 4b, 4b+1 = (lane t/4, columns 8b + 2(t%4), +1) and regs 4b+2, 4b+3 = the
// same columns of lane t/4 + 8 (profiles/r01_hw_microbench.txt, shape check)
__device__ __forceinline__ void lgp_tmem_ld16x256_x4(unsigned taddr, unsigned* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : LGP_R8(v, 0), LGP_R8(v, 8)
      : "r"(taddr));
}

// transposing FP64 reduction over lane bit o: lanes with the bit clear keep
// entries [0, h), the others [h, 2h); each half is summed with the partner's
template <int H>
__device__ __forceinline__ void lgp_xreduce(double* x, int o, bool up) {
#pragma unroll
  for (int m = 0; m < H; ++m) {
    const double send = up ? x[m] : x[m + H];
    const double keep = up ? x[m + H] : x[m];
    x[m] = keep + __shfl_xor_sync(0xffffffffu, send, o);
  }
}

extern "C" __global__ void __launch_bounds__(TS_THREADS, 1) lgp_matvec_tcsym(const LgpTcSymArgs a) {
  if (a.done != nullptr && *a.done) return;
  const int item = a.item_base + (int)blockIdx.x;
  const int I = a.items[3 * item], c0 = a.items[3 * item + 1], c1 = a.items[3 * item + 2];
  const int nch = c1 - c0;

  extern __shared__ __align__(1024) unsigned char ts_smem[];
  unsigned char* a1s = ts_smem;
  double* vis = reinterpret_cast<double*>(ts_smem + TC_A1_BYTES);  // p of the 128 rows
  unsigned char* stg = ts_smem + TC_A1_BYTES + 128 * 8;
  double* cbuf = reinterpret_cast<double*>(stg + LGP_TC_STAGES * TS_STAGE_BYTES);
  double* comb = cbuf + TS_CBUF_BYTES / 8;  // [NWG - 1][128] row sums of warpgroups 1..
  double* xpose = comb + 128 * (LGP_TS_NWG - 1);  // [epilogue warp][32 lanes][8] column transposes
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(xpose + TS_XPOSE_DOUBLES);
  unsigned* tslot = reinterpret_cast<unsigned*>(bars + TS_NBARS);
  const unsigned bar0 = lgp_saddr(bars);
#define TBAR(i) (bar0 + 8u * (unsigned)(i))

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    lgp_mbar_init(TBAR(TSB_AFULL), 1);
    for (int s = 0; s < LGP_TC_STAGES; ++s) {
      lgp_mbar_init(TBAR(TSB_SFULL(s)), 1);
      lgp_mbar_init(TBAR(TSB_SEMPTY(s)), 4);  // the 4 warps of the chunk's warpgroup
    }
    for (int q = 0; q < LGP_TS_NSB; ++q) {
      lgp_mbar_init(TBAR(TSB_S1FULL(q)), 1);
      lgp_mbar_init(TBAR(TSB_SFREE(q)), 4);
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
#define TS_SB(q) (tmem + 64u * (unsigned)(q))

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ producer (TMA bulk)
      lgp_mbar_expect_tx(TBAR(TSB_AFULL), TC_A1_BYTES + 128 * 8);
      lgp_bulk_g2s(lgp_saddr(a1s), a.a1 + (size_t)I * (TC_A1_BYTES / 4), TC_A1_BYTES,
                   TBAR(TSB_AFULL));
      lgp_bulk_g2s(lgp_saddr(vis), a.v + (size_t)I * 128, 128 * 8, TBAR(TSB_AFULL));
      for (int c = 0; c < nch; ++c) {
        const int s = c % LGP_TC_STAGES;
        if (c >= LGP_TC_STAGES) lgp_mbar_wait(TBAR(TSB_SEMPTY(s)), ((c / LGP_TC_STAGES) - 1) & 1);
        const unsigned dst = lgp_saddr(stg + (size_t)s * TS_STAGE_BYTES);
        lgp_mbar_expect_tx(TBAR(TSB_SFULL(s)), TS_STAGE_BYTES);
        lgp_bulk_g2s(dst,
                     reinterpret_cast<const unsigned char*>(a.b1) + (size_t)(c0 + c) * TC_B1_BYTES,
                     TC_B1_BYTES, TBAR(TSB_SFULL(s)));
        lgp_bulk_g2s(dst + TC_B1_BYTES, a.v + (size_t)(c0 + c) * TC_CH, TS_VCH_BYTES,
                     TBAR(TSB_SFULL(s)));
#if LGP_TC_PF
        lgp_bulk_g2s(dst + TC_B1_BYTES + TS_VCH_BYTES, a.c32 + (size_t)(c0 + c) * TC_CH * LGP_TC_FW,
                     TS_F32_BYTES, TBAR(TSB_SFULL(s)));
#endif
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------- distance-GEMM issuer
      const unsigned idesc1 = (1u << 4) | ((unsigned)(TC_CH >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
      const unsigned long long dk = lgp_sdesc(0u, LGP_TC_KD * 16);
      const unsigned long long a_d = dk + (lgp_saddr(a1s) >> 4);
      const unsigned stg0 = lgp_saddr(stg) >> 4;
      lgp_mbar_wait(TBAR(TSB_AFULL), 0);
      for (int c = 0; c < nch; ++c) {
        const int w = c % LGP_TS_NWG, k = c / LGP_TS_NWG;
        const int q = w + LGP_TS_NWG * (k % TS_NSBW);
        const int s = c % LGP_TC_STAGES;
        lgp_mbar_wait(TBAR(TSB_SFULL(s)), (c / LGP_TC_STAGES) & 1);
        if (k >= TS_NSBW) lgp_mbar_wait(TBAR(TSB_SFREE(q)), ((k / TS_NSBW) - 1) & 1);
        lgp_tc_fence_after();
        const unsigned long long b_d = dk + stg0 + (unsigned)s * (TS_STAGE_BYTES >> 4);
#pragma unroll
        for (int kk = 0; kk < LGP_TC_KD / 16; ++kk)
          lgp_mma_f16_ss(TS_SB(q), a_d + 16u * kk, b_d + 16u * kk, idesc1, kk > 0);
        lgp_mma_commit(TBAR(TSB_S1FULL(q)));
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------- epilogue warpgroups
#if LGP_TS_LAYOUT == 1
    // Each warp reads its 32 TMEM lanes as two 16x256b tiles per 32 columns:
    // thread t holds rows r0 + {0, 8, 16, 24} (r0 = t/4) x 8 columns
    // {8b + 2(t%4) + e}. The row side keeps 4 FP64 accumulators (reduced over
    // the 4 lanes of a row once per work item); the column side first sums its
    // 4 rows in registers, then a 3-level transposing butterfly over the 8
    // lanes sharing t%4 leaves one column per lane.
    const int w = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r0 = lane >> 2, cq = lane & 3;
    const int nloc = (nch - w + LGP_TS_NWG - 1) / LGP_TS_NWG;
    lgp_mbar_wait(TBAR(TSB_AFULL), 0);
    double vi[4], acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // u = 2h + v: row 32 q4 + 16 h + 8 v + r0
      vi[u] = vis[32 * q4 + 16 * (u >> 1) + 8 * (u & 1) + r0];
      acc[u] = 0.0;
    }
#if LGP_TC_PF && LGP_TS_RFG
    // Periodic features of the thread's 4 rows read through L1 at each use
    // (held in registers they spill: 96 registers at 4 warpgroups)
    const float* __restrict__ frb = a.r32 + (size_t)(128 * I + 32 * q4 + r0) * LGP_TC_FW + LGP_TC_P0;
#define TS_KJ(x, px, u, j) \
  lgp_tc_kf((x), a, (px), frb + (16 * ((u) >> 1) + 8 * ((u) & 1)) * LGP_TC_FW, cfp + (j) * LGP_TC_FW)
#elif LGP_TC_PF
    float frp[4][LGP_TC_PF];  // Periodic features of the thread's 4 rows
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int f = 0; f < LGP_TC_PF; ++f)
        frp[u][f] = a.r32[(size_t)(128 * I + 32 * q4 + 16 * (u >> 1) + 8 * (u & 1) + r0) * LGP_TC_FW +
                          LGP_TC_P0 + f];
#define TS_KJ(x, px, u, j) lgp_tc_kf((x), a, (px), frp[u], cfp + (j) * LGP_TC_FW)
#else
#define TS_KJ(x, px, u, j) lgp_tc_k((x), a, (px))
#endif
    // after the butterfly lane t holds column 8 k + 2 cq + e, k = 2 b4 + b3, e = b2
    const int ccol = 8 * (2 * ((lane >> 4) & 1) + ((lane >> 3) & 1)) + 2 * cq + ((lane >> 2) & 1);
    for (int k = 0; k < nloc; ++k) {
      const int c = LGP_TS_NWG * k + w;
      const int q = w + LGP_TS_NWG * (k % TS_NSBW);
      const int s = c % LGP_TC_STAGES;
      const int chunk = c0 + c;
      lgp_mbar_wait(TBAR(TSB_S1FULL(q)), (k / TS_NSBW) & 1);
      lgp_tc_fence_after();
      lgp_mbar_wait(TBAR(TSB_SFULL(s)), (c / LGP_TC_STAGES) & 1);  // p chunk visible
      const double* vj = reinterpret_cast<const double*>(stg + (size_t)s * TS_STAGE_BYTES + TC_B1_BYTES);
#if LGP_TC_PF
      const float* cfp = reinterpret_cast<const float*>(stg + (size_t)s * TS_STAGE_BYTES + TC_B1_BYTES +
                                                        TS_VCH_BYTES) + LGP_TC_P0;
#endif
      const bool diag = chunk < 2 * I + 2;
      // diagonal chunks: column offset relative to this thread's first row
      const int dj0 = chunk * TC_CH - (128 * I + 32 * q4 + r0) + 2 * cq;
      double* cb = cbuf + ((size_t)(w * 2 + (k & 1)) * 4 + q4) * TC_CH;
#if LGP_TS_PF
      // both 32-column halves in flight: the second half's TMEM latency hides
      // behind the first half's arithmetic
      unsigned svv[2][2][16];
      lgp_tmem_ld16x256_x4(TS_SB(q) + ((unsigned)(32 * q4) << 16), svv[0][0]);
      lgp_tmem_ld16x256_x4(TS_SB(q) + ((unsigned)(32 * q4 + 16) << 16), svv[0][1]);
      lgp_tmem_wait_ld();
      lgp_tmem_ld16x256_x4(TS_SB(q) + ((unsigned)(32 * q4) << 16) + 32u, svv[1][0]);
      lgp_tmem_ld16x256_x4(TS_SB(q) + ((unsigned)(32 * q4 + 16) << 16) + 32u, svv[1][1]);
#endif
#pragma unroll
      for (int g = 0; g < 2; ++g) {
#if LGP_TS_PF
        unsigned (&sv)[2][16] = svv[g];
        if (g == 1) {
          lgp_tmem_wait_ld();
          lgp_tc_fence_before();
          __syncwarp();
          if (lane == 0) lgp_mbar_arrive(TBAR(TSB_SFREE(q)));  // S buffer free for the next GEMM
        }
#else
        unsigned sv[2][16];
        lgp_tmem_ld16x256_x4(TS_SB(q) + ((unsigned)(32 * q4) << 16) + 32u * g, sv[0]);
        lgp_tmem_ld16x256_x4(TS_SB(q) + ((unsigned)(32 * q4 + 16) << 16) + 32u * g, sv[1]);
        lgp_tmem_wait_ld();
        if (g == 1) {
          lgp_tc_fence_before();
          __syncwarp();
          if (lane == 0) lgp_mbar_arrive(TBAR(TSB_SFREE(q)));  // S buffer free for the next GEMM
        }
#endif
        double pj[8];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double2 t2 = *reinterpret_cast<const double2*>(vj + 32 * g + 8 * b + 2 * cq);
          pj[2 * b] = t2.x;
          pj[2 * b + 1] = t2.y;
        }
        double cv[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) cv[m] = 0.0;
        // two separate unrolled loops: a per-entry diag test would cost a
        // branch + convergence barrier per entry (ncu: BSSY/BSYNC 17 % of issue)
        if (!diag) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 0; r < 16; ++r) {
              const int u = 2 * h + ((r >> 1) & 1), m = 2 * (r >> 2) + (r & 1);
#if (LGP_TS_ABLATE & 2)
              const double kd = lgp_widen_nn(__uint_as_float(sv[h][r]) * 0.5f);
#else
              const double kd = lgp_widen_nn(TS_KJ(LGP_TC_CLAMP(__uint_as_float(sv[h][r])),
                                                   r < LGP_TS_POLY ? 1 : 0, u,
                                                   32 * g + 8 * (r >> 2) + 2 * cq + (r & 1)));
#endif
              acc[u] = fma(kd, pj[m], acc[u]);
              cv[m] = fma(kd, vi[u], cv[m]);
            }
        } else {
          // diagonal block: row side j >= i, column side j > i
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 0; r < 16; ++r) {
              const int b = r >> 2, e = r & 1;
              const int u = 2 * h + ((r >> 1) & 1), m = 2 * b + e;
              const float kk = TS_KJ(LGP_TC_CLAMP(__uint_as_float(sv[h][r])), 0, u, 32 * g + 8 * b + 2 * cq + e);
              const int dj = dj0 + 32 * g + 8 * b + e - (16 * h + 8 * ((r >> 1) & 1));  // j - i
              acc[u] = fma(lgp_widen_nn(dj >= 0 ? kk : 0.f), pj[m], acc[u]);
              cv[m] = fma(lgp_widen_nn(dj > 0 ? kk : 0.f), vi[u], cv[m]);
            }
        }
#if (LGP_TS_ABLATE & 1)  // timing diagnostics only (wrong results)
        cb[32 * g + ccol] = ((cv[0] + cv[1]) + (cv[2] + cv[3])) + ((cv[4] + cv[5]) + (cv[6] + cv[7]));
#elif LGP_TS_XPOSE
        {
          // lane t stores its 8 column partials as 4 x 16 B (pair position
          // swizzled by (t >> 1) & 3: conflict-free), then lane l sums slot
          // l >> 2 of the 8 lanes sharing its column group, rows in order
          // (4 STS.128 + 8 LDS.64 + 7 DADD per 32 entries; the butterfly
          // needed 14 SHFL + 28 FSEL + 7 DADD)
          double* xw = xpose + (size_t)(warp - 2) * 32 * 8;
          const int sw = (lane >> 1) & 3;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            *reinterpret_cast<double2*>(xw + lane * 8 + 2 * (i ^ sw)) = make_double2(cv[2 * i], cv[2 * i + 1]);
          __syncwarp();
          const int mm = lane >> 2;
          double col = 0.0;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int tt = 4 * r + cq;
            col += xw[tt * 8 + 2 * ((mm >> 1) ^ ((tt >> 1) & 3)) + (mm & 1)];
          }
          __syncwarp();  // the next half overwrites xw
          cb[32 * g + ccol] = col;
        }
#else
        lgp_xreduce<4>(cv, 16, (lane & 16) != 0);
        lgp_xreduce<2>(cv, 8, (lane & 8) != 0);
        lgp_xreduce<1>(cv, 4, (lane & 4) != 0);
        cb[32 * g + ccol] = cv[0];
#endif
      }
      __syncwarp();
      if (lane == 0) lgp_mbar_arrive(TBAR(TSB_SEMPTY(s)));  // p chunk read: stage reusable
#if !(LGP_TS_ABLATE & 4)
      asm volatile("bar.sync %0, 128;" ::"r"(1 + w) : "memory");
#endif
      // column partials of this (I, chunk): warps 0..3 in a fixed order
      if (lane < 16) {
        const int j = 16 * q4 + lane;
        const double* b0 = cbuf + (size_t)(w * 2 + (k & 1)) * 4 * TC_CH;
        const double sum = ((b0[j] + b0[TC_CH + j]) + b0[2 * TC_CH + j]) + b0[3 * TC_CH + j];
        a.colpart[(size_t)(a.colbase[I] + chunk - 2 * I) * TC_CH + j] = sum;
      }
    }
    // row side: the 4 lanes of a row (lane bits 0, 1) -> lane holds u = 2 b1 + b0
    lgp_xreduce<2>(acc, 2, (lane & 2) != 0);
    lgp_xreduce<1>(acc, 1, (lane & 1) != 0);
    const int ur = 2 * ((lane >> 1) & 1) + (lane & 1);
    const int row = 32 * q4 + 16 * (ur >> 1) + 8 * (ur & 1) + r0;
    if (w > 0) comb[(w - 1) * 128 + row] = acc[0];
    asm volatile("bar.sync %0, %1;" ::"r"(LGP_TS_NWG + 1), "r"(128 * LGP_TS_NWG) : "memory");
    if (w == 0) {
      double r = acc[0];
#pragma unroll
      for (int u = 1; u < LGP_TS_NWG; ++u) r += comb[(u - 1) * 128 + row];
      a.rowpart[(size_t)item * 128 + row] = r;
    }
#else
    const int w = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int row = 32 * q4 + lane;
    const unsigned lanes = (unsigned)(32 * q4) << 16;
    const int nloc = (nch - w + LGP_TS_NWG - 1) / LGP_TS_NWG;
    const long long gi = 128ll * I + row;
    lgp_mbar_wait(TBAR(TSB_AFULL), 0);
    const double vi = vis[row];
    double acc = 0.0;
    for (int k = 0; k < nloc; ++k) {
      const int c = LGP_TS_NWG * k + w;
      const int q = w + LGP_TS_NWG * (k % TS_NSBW);
      const int s = c % LGP_TC_STAGES;
      const int chunk = c0 + c;
      lgp_mbar_wait(TBAR(TSB_S1FULL(q)), (k / TS_NSBW) & 1);
      lgp_tc_fence_after();
      lgp_mbar_wait(TBAR(TSB_SFULL(s)), (c / LGP_TC_STAGES) & 1);  // p chunk visible
      const double* vj = reinterpret_cast<const double*>(stg + (size_t)s * TS_STAGE_BYTES + TC_B1_BYTES);
      // columns of this chunk intersect the row block's diagonal: mask
      const bool diag = chunk < 2 * I + 2;
      const long long gj0 = (long long)chunk * TC_CH;
      double* cb = cbuf + ((size_t)(w * 2 + (k & 1)) * 4 + q4) * TC_CH;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        // 32 columns per round trip (register budget of 3 warpgroups)
        unsigned sv[32];
        lgp_tmem_ld32p(TS_SB(q) + lanes + 32u * g, sv);
        lgp_tmem_wait_ld();
        if (g == 1) {
          lgp_tc_fence_before();
          __syncwarp();
          if (lane == 0) lgp_mbar_arrive(TBAR(TSB_SFREE(q)));  // S buffer free for the next GEMM
        }
        double cv[32];
        if (!diag) {
          // off-diagonal chunk: every entry feeds both sides
#pragma unroll
          for (int m = 0; m < 32; ++m) {
            const int j = 32 * g + m;
            const double kd = lgp_widen_nn(lgp_tc_k(LGP_TC_CLAMP(__uint_as_float(sv[m])), a, 0));
            acc = fma(kd, vj[j], acc);
            cv[m] = kd * vi;
          }
        } else {
          // diagonal block: row side j >= i, column side j > i
#pragma unroll
          for (int m = 0; m < 32; ++m) {
            const int j = 32 * g + m;
            const long long gj = gj0 + j;
            const float kk = lgp_tc_k(LGP_TC_CLAMP(__uint_as_float(sv[m])), a, 0);
            acc = fma(lgp_widen_nn(gj >= gi ? kk : 0.f), vj[j], acc);
            cv[m] = lgp_widen_nn(gj > gi ? kk : 0.f) * vi;
          }
        }
        // transpose-reduce over the warp: after level o each lane keeps o
        // partial columns; after 5 levels lane l holds column 32g + l
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int m = 0; m < o; ++m) {
            const double send = up ? cv[m] : cv[m + o];
            const double keep = up ? cv[m + o] : cv[m];
            cv[m] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        cb[32 * g + lane] = cv[0];
      }
      __syncwarp();
      if (lane == 0) lgp_mbar_arrive(TBAR(TSB_SEMPTY(s)));  // p chunk read: stage reusable
      asm volatile("bar.sync %0, 128;" ::"r"(1 + w) : "memory");
      // column partials of this (I, chunk): warps 0..3 in a fixed order
      if (lane < 16) {
        const int j = 16 * q4 + lane;
        const double* b0 = cbuf + (size_t)(w * 2 + (k & 1)) * 4 * TC_CH;
        const double sum = ((b0[j] + b0[TC_CH + j]) + b0[2 * TC_CH + j]) + b0[3 * TC_CH + j];
        a.colpart[(size_t)(a.colbase[I] + chunk - 2 * I) * TC_CH + j] = sum;
      }
    }
    // row partial of this segment: warpgroups 0, 1, .. in a fixed order
    if (w > 0) comb[(w - 1) * 128 + row] = acc;
    asm volatile("bar.sync %0, %1;" ::"r"(LGP_TS_NWG + 1), "r"(128 * LGP_TS_NWG) : "memory");
    if (w == 0) {
      double r = acc;
#pragma unroll
      for (int u = 1; u < LGP_TS_NWG; ++u) r += comb[(u - 1) * 128 + row];
      a.rowpart[(size_t)item * 128 + row] = r;
    }
#endif
  }
  lgp_tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    lgp_tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
#undef TBAR
#undef TS_SB
}

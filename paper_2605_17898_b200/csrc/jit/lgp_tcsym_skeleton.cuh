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
//     DFMA per entry in the row's thread, the column side k_ij * p_i is summed
//     over the thread's 4 rows and reduced over the lanes / warps sharing a
//     column in a fixed order.
// Diagonal tiles: entries j > i go to both sides, j == i to the row side only,
// j < i are skipped (they are the pair's other orientation).
//
// Work item = one rectangle of the (row block I, chunk c) triangle (c >= 2I):
// row blocks [Ia, Ib) x chunks [ca, cb), at most R x 2R - the host tiles the
// triangle with R x 2R super-tiles and splits the ones dispatched last into
// quarters (load balance of the final wave). Rows run outer, chunks inner;
// inside the CTA
//   * column partials accumulate in shared memory over the item's row blocks,
//     one accumulator per (warp, chunk, column) so no warp waits for another
//     (each chunk owned by one epilogue warpgroup, rows in order; the 4 warps
//     combined in a fixed order once per item), and
//   * row partials of the 4 warpgroups are combined per row block by a
//     combiner warp (warpgroups in order),
// so the item writes R x 128 row and 2R x 64 column FP64 partials once:
// O(items x R) scratch, with R chosen per operator so that the item count
// (and with it the scratch, ~N x const) stays a few waves of the GPU. The
// epilogue kernel sums each row block's / chunk's records in a fixed order
// (deterministic).
//
// Warps: 0 producer (cp.async.bulk: row tile + p rows per row block, ring of
// column-feature tiles + p chunks), 1 distance-GEMM issuer, 2.. LGP_TS_NWG
// epilogue warpgroups (chunk c -> warpgroup (c - ca) % NWG). (A dedicated
// row-combiner warp cost the epilogue 16 registers per thread: 2.47 vs 2.33 ms
// at cfg4.)

#ifndef LGP_TS_NWG
#define LGP_TS_NWG 4  // epilogue warpgroups: latency hiding
#endif
#define TS_THREADS (64 + 128 * LGP_TS_NWG)
#define LGP_TS_NSB 8                     // S buffers of 64 TMEM columns (all 512)
#define TS_NSBW (LGP_TS_NSB / LGP_TS_NWG)  // S buffers per warpgroup
#define TS_VCH_BYTES (TC_CH * 8)           // p chunk, FP64
#define TS_F32_BYTES (LGP_TC_PF ? TC_CH * LGP_TC_FW * 4 : 0)  // column Periodic features
#define TS_STAGE_BYTES (TC_B1_BYTES + TS_VCH_BYTES + TS_F32_BYTES)
#define TS_A_BYTES (TC_A1_BYTES + 128 * 8)  // row tile + p of its 128 rows
#define TS_RBUF_DOUBLES (LGP_TS_NWG * 2 * 128)        // [wg][slot][128]
#define TS_NBARS (10 + 2 * LGP_TC_STAGES + 2 * LGP_TS_NSB)  // (incl. 2 ticket counters)
#define TS_NA 3  // row-tile buffers: row u + 2 loads while row u computes
#define TSB_AFULL(b) (b)
#define TSB_AEMPTY(b) (TS_NA + (b))
#define TSB_RCNT(b) (2 * TS_NA + (b))  // not an mbarrier: ticket counter of the row deposits
#define TSB_RFREE(b) (2 * TS_NA + 2 + (b))
#define TSB_SFULL(s) (2 * TS_NA + 4 + (s))
#define TSB_SEMPTY(s) (2 * TS_NA + 4 + LGP_TC_STAGES + (s))
#define TSB_S1FULL(q) (2 * TS_NA + 4 + 2 * LGP_TC_STAGES + (q))
#define TSB_SFREE(q) (2 * TS_NA + 4 + 2 * LGP_TC_STAGES + LGP_TS_NSB + (q))
// shared memory: [TS_NA][TS_A_BYTES] | stages | rbuf | bars | tslot | colacc [4][2R][64]
#define TS_SMEM_FIXED \
  (TS_NA * TS_A_BYTES + LGP_TC_STAGES * TS_STAGE_BYTES + 8 * (TS_RBUF_DOUBLES + TS_NBARS) + 16)

// FP32 -> FP64 for finite non-negative kernel values without the conversion
// pipe (F2F.F64.F32 runs at 16/clk/SM): exponent re-bias + mantissa shift
// (0 maps to 2^-127, negligible). (Keeping the FP32 pattern as the low word,
// one op instead of two, measured slower: 2.47 vs 2.39 ms at cfg4.)
__device__ __forceinline__ double lgp_widen_nn(float f) {
  const unsigned b = __float_as_uint(f);
  return __hiloint2double((b >> 3) + 0x38000000u, b << 29);
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
  const int I0 = a.items[6 * item], I1 = a.items[6 * item + 1];
  const int c_lo = a.items[6 * item + 2], c_hi = a.items[6 * item + 3];
  // this item's first row / chunk record (relative to the launch's first item)
  const int rrec = a.items[6 * item + 4] - a.items[6 * a.item_base + 4];
  const int crec = a.items[6 * item + 5] - a.items[6 * a.item_base + 5];
  // first chunk of row block I: the pair's max is in chunk >= 2I
#define TS_CS(I) max(c_lo, 2 * (I))

  extern __shared__ __align__(1024) unsigned char ts_smem[];
  unsigned char* abuf = ts_smem;  // [TS_NA][row tile | p rows]
  unsigned char* stg = ts_smem + TS_NA * TS_A_BYTES;
  double* rbuf = reinterpret_cast<double*>(stg + LGP_TC_STAGES * TS_STAGE_BYTES);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(rbuf + TS_RBUF_DOUBLES);
  unsigned* tslot = reinterpret_cast<unsigned*>(bars + TS_NBARS);
  double* colacc = reinterpret_cast<double*>(ts_smem + TS_SMEM_FIXED);  // [warp][2R][64]
  const int CM = 2 * a.R;  // chunks per item at most
  const unsigned bar0 = lgp_saddr(bars);
#define TBAR(i) (bar0 + 8u * (unsigned)(i))

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    for (int b = 0; b < TS_NA; ++b) {
      lgp_mbar_init(TBAR(TSB_AFULL(b)), 1);
      lgp_mbar_init(TBAR(TSB_AEMPTY(b)), 1 + 4 * LGP_TS_NWG);  // last MMA of the row + epilogue warps
    }
    for (int b = 0; b < 2; ++b) {
      bars[TSB_RCNT(b)] = 0ull;
      lgp_mbar_init(TBAR(TSB_RFREE(b)), 1);
    }
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
      // row tile + p rows of row u + 2 go out once row u's chunks are queued
      auto load_a = [&](int u) {
        const int b = u % TS_NA, I = I0 + u;
        if (u >= TS_NA) lgp_mbar_wait(TBAR(TSB_AEMPTY(b)), ((u / TS_NA) - 1) & 1);
        unsigned char* ab = abuf + (size_t)b * TS_A_BYTES;
        lgp_mbar_expect_tx(TBAR(TSB_AFULL(b)), TS_A_BYTES);
        lgp_bulk_g2s(lgp_saddr(ab), a.a1 + (size_t)I * (TC_A1_BYTES / 4), TC_A1_BYTES, TBAR(TSB_AFULL(b)));
        lgp_bulk_g2s(lgp_saddr(ab + TC_A1_BYTES), a.v + (size_t)I * 128, 128 * 8, TBAR(TSB_AFULL(b)));
      };
      for (int u = 0; u < 2 && I0 + u < I1; ++u) load_a(u);
      int f = 0;
      for (int I = I0; I < I1; ++I) {
        for (int c = TS_CS(I); c < c_hi; ++c, ++f) {
          const int s = f % LGP_TC_STAGES;
          if (f >= LGP_TC_STAGES) lgp_mbar_wait(TBAR(TSB_SEMPTY(s)), ((f / LGP_TC_STAGES) - 1) & 1);
          const unsigned dst = lgp_saddr(stg + (size_t)s * TS_STAGE_BYTES);
          lgp_mbar_expect_tx(TBAR(TSB_SFULL(s)), TS_STAGE_BYTES);
          lgp_bulk_g2s(dst, reinterpret_cast<const unsigned char*>(a.b1) + (size_t)c * TC_B1_BYTES,
                       TC_B1_BYTES, TBAR(TSB_SFULL(s)));
          lgp_bulk_g2s(dst + TC_B1_BYTES, a.v + (size_t)c * TC_CH, TS_VCH_BYTES, TBAR(TSB_SFULL(s)));
#if LGP_TC_PF
          lgp_bulk_g2s(dst + TC_B1_BYTES + TS_VCH_BYTES, a.c32 + (size_t)c * TC_CH * LGP_TC_FW,
                       TS_F32_BYTES, TBAR(TSB_SFULL(s)));
#endif
        }
        if (I + 2 < I1) load_a(I + 2 - I0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------- distance-GEMM issuer
      const unsigned idesc1 = (1u << 4) | ((unsigned)(TC_CH >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
      const unsigned long long dk = lgp_sdesc(0u, LGP_TC_KD * 16);
      const unsigned stg0 = lgp_saddr(stg) >> 4;
      int f = 0;
      int kw[LGP_TS_NWG];
#pragma unroll
      for (int w = 0; w < LGP_TS_NWG; ++w) kw[w] = 0;
      for (int I = I0; I < I1; ++I) {
        const int u = I - I0, b = u % TS_NA;
        const unsigned long long a_d = dk + (lgp_saddr(abuf + (size_t)b * TS_A_BYTES) >> 4);
        lgp_mbar_wait(TBAR(TSB_AFULL(b)), (u / TS_NA) & 1);
        const int cs = TS_CS(I);
        for (int c = cs; c < c_hi; ++c, ++f) {
          const int w = (c - c_lo) % LGP_TS_NWG;
          int k = 0;
#pragma unroll
          for (int x = 0; x < LGP_TS_NWG; ++x)
            if (x == w) k = kw[x]++;
          const int q = w + LGP_TS_NWG * (k % TS_NSBW);
          const int s = f % LGP_TC_STAGES;
          lgp_mbar_wait(TBAR(TSB_SFULL(s)), (f / LGP_TC_STAGES) & 1);
          if (k >= TS_NSBW) lgp_mbar_wait(TBAR(TSB_SFREE(q)), ((k / TS_NSBW) - 1) & 1);
          lgp_tc_fence_after();
          const unsigned long long b_d = dk + stg0 + (unsigned)s * (TS_STAGE_BYTES >> 4);
#pragma unroll
          for (int kk = 0; kk < LGP_TC_KD / 16; ++kk)
            lgp_mma_f16_ss(TS_SB(q), a_d + 16u * kk, b_d + 16u * kk, idesc1, kk > 0);
          lgp_mma_commit(TBAR(TSB_S1FULL(q)));
        }
        lgp_mma_commit(TBAR(TSB_AEMPTY(b)));  // this row tile is no longer read
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------- epilogue warpgroups
    // Each warp reads its 32 TMEM lanes as two 16x256b tiles per 32 columns:
    // thread t holds rows r0 + {0, 8, 16, 24} (r0 = t/4) x 8 columns
    // {8b + 2(t%4) + e}. The row side keeps 4 FP64 accumulators (reduced over
    // the 4 lanes of a row at the end of each row block); the column side
    // first sums its 4 rows in registers, then a 3-level transposing
    // butterfly over the 8 lanes sharing t%4 leaves one column per lane.
    const int w = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r0 = lane >> 2, cq = lane & 3;
    // after the butterfly lane t holds column 8 k + 2 cq + e, k = 2 b4 + b3, e = b2
    const int ccol = 8 * (2 * ((lane >> 4) & 1) + ((lane >> 3) & 1)) + 2 * cq + ((lane >> 2) & 1);
    // this warp's column accumulators of the warpgroup's chunks: entries
    // (q4, c, 32 g + ccol) belong to this lane alone, row blocks in order
    double* cacc = colacc + (size_t)q4 * CM * TC_CH + ccol;
    for (int c = c_lo + w; c < c_hi; c += LGP_TS_NWG) {
      cacc[(size_t)(c - c_lo) * TC_CH] = 0.0;
      cacc[(size_t)(c - c_lo) * TC_CH + 32] = 0.0;
    }
    int f_row = 0;  // flat chunk index of the row block's first chunk
    int k = 0;      // this warpgroup's chunk counter
    for (int I = I0; I < I1; ++I) {
      const int u = I - I0, b = u & 1, ba = u % TS_NA;
      lgp_mbar_wait(TBAR(TSB_AFULL(ba)), (u / TS_NA) & 1);
      const double* vis = reinterpret_cast<const double*>(abuf + (size_t)ba * TS_A_BYTES + TC_A1_BYTES);
      double vi[4], acc[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {  // x = 2h + v: row 32 q4 + 16 h + 8 v + r0
        vi[x] = vis[32 * q4 + 16 * (x >> 1) + 8 * (x & 1) + r0];
        acc[x] = 0.0;
      }
      __syncwarp();
      if (lane == 0) lgp_mbar_arrive(TBAR(TSB_AEMPTY(ba)));  // p rows read
#if LGP_TC_PF
      float frp[4][LGP_TC_PF];  // Periodic features of the thread's 4 rows
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int f = 0; f < LGP_TC_PF; ++f)
          frp[x][f] = a.r32[(size_t)(128 * I + 32 * q4 + 16 * (x >> 1) + 8 * (x & 1) + r0) * LGP_TC_FW +
                            LGP_TC_P0 + f];
#define TS_KJ(x, px, u, j) lgp_tc_kf((x), a, (px), frp[u], cfp + (j) * LGP_TC_FW)
#else
#define TS_KJ(x, px, u, j) lgp_tc_k((x), a, (px))
#endif
      const int cs = TS_CS(I);
      // this warpgroup's first chunk of the row: c = c_lo + w (mod NWG)
      const int c_first = cs + (((w - (cs - c_lo)) % LGP_TS_NWG) + LGP_TS_NWG) % LGP_TS_NWG;
      const bool dblk = cs < 2 * I + 2;  // the row block's diagonal chunks are in this item
      for (int c = c_first; c < c_hi; c += LGP_TS_NWG, ++k) {
        const int f = f_row + (c - cs);
        const int q = w + LGP_TS_NWG * (k % TS_NSBW);
        const int s = f % LGP_TC_STAGES;
        lgp_mbar_wait(TBAR(TSB_S1FULL(q)), (k / TS_NSBW) & 1);
        lgp_tc_fence_after();
        lgp_mbar_wait(TBAR(TSB_SFULL(s)), (f / LGP_TC_STAGES) & 1);  // p chunk visible
        const double* vj = reinterpret_cast<const double*>(stg + (size_t)s * TS_STAGE_BYTES + TC_B1_BYTES);
#if LGP_TC_PF
        const float* cfp = reinterpret_cast<const float*>(stg + (size_t)s * TS_STAGE_BYTES + TC_B1_BYTES +
                                                          TS_VCH_BYTES) + LGP_TC_P0;
#endif
        const bool diag = dblk && c < 2 * I + 2;
        // diagonal chunks: column offset relative to this thread's first row
        const int dj0 = c * TC_CH - (128 * I + 32 * q4 + r0) + 2 * cq;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          unsigned sv[2][16];
          lgp_tmem_ld16x256_x4(TS_SB(q) + ((unsigned)(32 * q4) << 16) + 32u * g, sv[0]);
          lgp_tmem_ld16x256_x4(TS_SB(q) + ((unsigned)(32 * q4 + 16) << 16) + 32u * g, sv[1]);
          lgp_tmem_wait_ld();
          if (g == 1) {
            lgp_tc_fence_before();
            __syncwarp();
            if (lane == 0) lgp_mbar_arrive(TBAR(TSB_SFREE(q)));  // S buffer free for the next GEMM
          }
          double pj[8];
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const double2 t2 = *reinterpret_cast<const double2*>(vj + 32 * g + 8 * bb + 2 * cq);
            pj[2 * bb] = t2.x;
            pj[2 * bb + 1] = t2.y;
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
                const int x = 2 * h + ((r >> 1) & 1), m = 2 * (r >> 2) + (r & 1);
                const double kd = lgp_widen_nn(TS_KJ(LGP_TC_CLAMP(__uint_as_float(sv[h][r])), 0, x,
                                                     32 * g + 8 * (r >> 2) + 2 * cq + (r & 1)));
                acc[x] = fma(kd, pj[m], acc[x]);
                cv[m] = fma(kd, vi[x], cv[m]);
              }
          } else {
            // diagonal block: row side j >= i, column side j > i
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int r = 0; r < 16; ++r) {
                const int bb = r >> 2, e = r & 1;
                const int x = 2 * h + ((r >> 1) & 1), m = 2 * bb + e;
                const float kk = TS_KJ(LGP_TC_CLAMP(__uint_as_float(sv[h][r])), 0, x, 32 * g + 8 * bb + 2 * cq + e);
                const int dj = dj0 + 32 * g + 8 * bb + e - (16 * h + 8 * ((r >> 1) & 1));  // j - i
                acc[x] = fma(lgp_widen_nn(dj >= 0 ? kk : 0.f), pj[m], acc[x]);
                cv[m] = fma(lgp_widen_nn(dj > 0 ? kk : 0.f), vi[x], cv[m]);
              }
          }
          lgp_xreduce<4>(cv, 16, (lane & 16) != 0);
          lgp_xreduce<2>(cv, 8, (lane & 8) != 0);
          lgp_xreduce<1>(cv, 4, (lane & 4) != 0);
          cacc[(size_t)(c - c_lo) * TC_CH + 32 * g] += cv[0];
        }
        __syncwarp();
        if (lane == 0) lgp_mbar_arrive(TBAR(TSB_SEMPTY(s)));  // p chunk read: stage reusable
      }
      f_row += c_hi - cs;
      // row side: the 4 lanes of a row (lane bits 0, 1) -> lane holds x = 2 b1 + b0
      lgp_xreduce<2>(acc, 2, (lane & 2) != 0);
      lgp_xreduce<1>(acc, 1, (lane & 1) != 0);
      const int xr = 2 * ((lane >> 1) & 1) + (lane & 1);
      const int row = 32 * q4 + 16 * (xr >> 1) + 8 * (xr & 1) + r0;
      if (u >= 2) lgp_mbar_wait(TBAR(TSB_RFREE(b)), ((u >> 1) - 1) & 1);
      rbuf[(w * 2 + b) * 128 + row] = acc[0];
      __syncwarp();
      // the last of the 4 NWG warps to deposit sums the row block's partial
      // (warpgroups in order) and frees the slot
      unsigned last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(reinterpret_cast<unsigned*>(&bars[TSB_RCNT(b)]), 1u) == 4u * LGP_TS_NWG - 1u;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence_block();
        double* rp = a.rowpart + ((size_t)rrec + u) * 128;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int rr = lane + 32 * m;
          double sum = rbuf[b * 128 + rr];
#pragma unroll
          for (int x = 1; x < LGP_TS_NWG; ++x) sum += rbuf[(x * 2 + b) * 128 + rr];
          rp[rr] = sum;
        }
        __syncwarp();
        if (lane == 0) {
          *reinterpret_cast<volatile unsigned*>(&bars[TSB_RCNT(b)]) = 0u;
          lgp_mbar_arrive(TBAR(TSB_RFREE(b)));
        }
      }
#undef TS_KJ
    }
    // the item's column partials: the warpgroup's 4 warps in a fixed order
    asm volatile("bar.sync %0, 128;" ::"r"(1 + w) : "memory");
    if (lane < 16) {
      const int j = 16 * q4 + lane;
      double* cp = a.colpart + (size_t)crec * TC_CH;
      for (int c = c_lo + w; c < c_hi; c += LGP_TS_NWG) {
        const double* ca = colacc + (size_t)(c - c_lo) * TC_CH + j;
        cp[(size_t)(c - c_lo) * TC_CH + j] =
            ((ca[0] + ca[(size_t)CM * TC_CH]) + ca[(size_t)2 * CM * TC_CH]) + ca[(size_t)3 * CM * TC_CH];
      }
    }
  }
  lgp_tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    lgp_tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
#undef TS_CS
#undef TBAR
#undef TS_SB
}

// K1-TC v5 (lgp_matvec_tc4): the distance tile on warp-level mma.sync in the
// epilogue warps, many epilogue warpgroups. Appended after lgp_tc_skeleton.cuh
// (helpers, feature tiles, generated lgp_tc_k), single CTA (no pairs).
//
// The v4 kernel (lgp_matvec_tc) is bound by tcgen05.ld of the FP32 -r^2 tile
// (40.8 B/clk/SM, 4 B per entry). Here each epilogue warp computes -r^2 of its
// 32 rows x 64 columns with mma.sync m16n8k16 (A = row features in shared
// memory, B = the staged column features, both via ldmatrix from the UMMA
// K-major layout), so -r^2 never leaves registers; the tree, the FP16 hi/lo
// split and a tcgen05.st in the accumulator layout (16x128b) follow, and the
// contraction stays on tcgen05 (A = P from TMEM). NWG epilogue warpgroups take
// chunks round-robin so one warp's mma.sync phase overlaps another's MUFU
// phase. FP64 per-row sums live in shared memory (registers are scarce).
//
// Warps: 0 producer (TMA ring of column features + V tiles), 1 / 2 contraction
// issuers (warpgroups w = 0, 2, .. / 1, 3, ..; chunks in order), 3.. epilogue.
// TMEM: P buffer of warpgroup w at 64 w, its two D2 accumulators after them.

#ifndef LGP_T4_NWG
#define LGP_T4_NWG 4
#endif
#define T4_THREADS (96 + 128 * LGP_T4_NWG)
#define T4_NBARS (1 + 2 * LGP_TC_STAGES + 2 * LGP_T4_NWG + 4 * LGP_T4_NWG)
#define T4B_AFULL 0
#define T4B_SFULL(s) (1 + (s))
#define T4B_SEMPTY(s) (1 + LGP_TC_STAGES + (s))
#define T4B_PFULL(w) (1 + 2 * LGP_TC_STAGES + (w))
#define T4B_PEMPTY(w) (1 + 2 * LGP_TC_STAGES + LGP_T4_NWG + (w))
#define T4B_D2FULL(w, b) (1 + 2 * LGP_TC_STAGES + 2 * LGP_T4_NWG + 2 * (w) + (b))
#define T4B_D2EMPTY(w, b) (1 + 2 * LGP_TC_STAGES + 4 * LGP_T4_NWG + 2 * (w) + (b))
#if 64 * LGP_T4_NWG + 2 * TC_N2 * LGP_T4_NWG > 512
#error "TMEM budget of lgp_matvec_tc4"
#endif

#if !LGP_TC_PAIR
extern "C" __global__ void __launch_bounds__(T4_THREADS, 1) lgp_matvec_tc4(const LgpTcArgs a) {
  if (a.done != nullptr && *a.done) return;
  const int rb = blockIdx.x % a.n_rb;
  const int rest = blockIdx.x / a.n_rb;
  const int seg = rest % a.n_seg;
  const int pass = rest / a.n_seg;
  const int tile0 = seg * a.tiles_per_seg;
  int nch = a.n_tiles - tile0;
  if (nch > a.tiles_per_seg) nch = a.tiles_per_seg;

  extern __shared__ __align__(1024) unsigned char t4_smem[];
  unsigned char* a1s = t4_smem;
  unsigned char* stg = t4_smem + TC_A1_BYTES;
  double* accs = reinterpret_cast<double*>(stg + LGP_TC_STAGES * TC_STAGE_BYTES);  // [NWG][N][128]
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(accs + (size_t)LGP_T4_NWG * LGP_TC_N * 128);
  unsigned* tslot = reinterpret_cast<unsigned*>(bars + T4_NBARS);
  const unsigned bar0 = lgp_saddr(bars);
#define TB4(i) (bar0 + 8u * (unsigned)(i))

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  if (tid == 0) {
    lgp_mbar_init(TB4(T4B_AFULL), 1);
    for (int s = 0; s < LGP_TC_STAGES; ++s) {
      lgp_mbar_init(TB4(T4B_SFULL(s)), 1);
      lgp_mbar_init(TB4(T4B_SEMPTY(s)), 1);
    }
    for (int w = 0; w < LGP_T4_NWG; ++w) {
      lgp_mbar_init(TB4(T4B_PFULL(w)), 4);
      lgp_mbar_init(TB4(T4B_PEMPTY(w)), 1);
      for (int b = 0; b < 2; ++b) {
        lgp_mbar_init(TB4(T4B_D2FULL(w, b)), 1);
        lgp_mbar_init(TB4(T4B_D2EMPTY(w, b)), 4);
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
#define T4_P(w) (tmem + 64u * (unsigned)(w))
#define T4_D2(w, b) (tmem + 64u * LGP_T4_NWG + (unsigned)TC_N2 * (2u * (unsigned)(w) + (unsigned)(b)))
  const unsigned stg0 = lgp_saddr(stg) >> 4;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ producer (TMA bulk)
      lgp_mbar_expect_tx(TB4(T4B_AFULL), TC_A1_BYTES);
      lgp_bulk_g2s(lgp_saddr(a1s), a.a1 + (size_t)rb * (TC_A1_BYTES / 4), TC_A1_BYTES,
                   TB4(T4B_AFULL));
      const unsigned char* vbase = reinterpret_cast<const unsigned char*>(a.v);
      for (int c = 0; c < nch; ++c) {
        const int s = c % LGP_TC_STAGES;
        if (c >= LGP_TC_STAGES) lgp_mbar_wait(TB4(T4B_SEMPTY(s)), ((c / LGP_TC_STAGES) - 1) & 1);
        const unsigned dst = lgp_saddr(stg + (size_t)s * TC_STAGE_BYTES);
        lgp_mbar_expect_tx(TB4(T4B_SFULL(s)), TC_B1_BYTES + TC_V_BYTES);
        lgp_bulk_g2s(dst, reinterpret_cast<const unsigned char*>(a.b1) + (size_t)(tile0 + c) * TC_B1_BYTES,
                     TC_B1_BYTES, TB4(T4B_SFULL(s)));
        lgp_bulk_g2s(dst + TC_B1_BYTES, vbase + ((size_t)pass * a.n_tiles + tile0 + c) * TC_V_BYTES,
                     TC_V_BYTES, TB4(T4B_SFULL(s)));
      }
    }
    __syncwarp();
  } else if (warp == 1 || warp == 2) {
    if (lane == 0) {
      // --------------------------------------- contraction issuers (tcgen05)
      // issuer j takes the chunks of warpgroups w = j, j + 2, .. in chunk order
      const unsigned idesc2 = (1u << 4) | ((unsigned)(TC_N2 >> 3) << 17) | ((unsigned)(128 >> 4) << 24);
      const unsigned long long dv = lgp_sdesc(0u, 1024u);
      for (int c = 0; c < nch; ++c) {
        const int w = c % LGP_T4_NWG, k = c / LGP_T4_NWG;  // k-th chunk of warpgroup w
        if ((w & 1) != warp - 1) continue;
        const int gi = k / LGP_TC_G, b = gi & 1;
        const int nloc = (nch - w + LGP_T4_NWG - 1) / LGP_T4_NWG;
        const bool first = (k % LGP_TC_G) == 0;
        const bool last = ((k % LGP_TC_G) == LGP_TC_G - 1) || (k == nloc - 1);
        lgp_mbar_wait(TB4(T4B_PFULL(w)), k & 1);
        if (first && gi >= 2) lgp_mbar_wait(TB4(T4B_D2EMPTY(w, b)), ((gi >> 1) - 1) & 1);
        lgp_tc_fence_after();
        const int s = c % LGP_TC_STAGES;
        const unsigned long long v_d = dv + stg0 + (unsigned)s * (TC_STAGE_BYTES >> 4) + (TC_B1_BYTES >> 4);
        const unsigned d = T4_D2(w, b), p = T4_P(w);
#pragma unroll
        for (int kk = 0; kk < TC_CH / 16; ++kk) {
          lgp_mma_f16_ts(d, p + 8u * kk, v_d + 16u * kk, idesc2, (first && kk == 0) ? 0u : 1u);
          lgp_mma_f16_ts(d, p + 32u + 8u * kk, v_d + 16u * kk, idesc2, 1u);
        }
        lgp_mma_commit(TB4(T4B_SEMPTY(s)));
        lgp_mma_commit(TB4(T4B_PEMPTY(w)));
        if (last) lgp_mma_commit(TB4(T4B_D2FULL(w, b)));
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------- epilogue warpgroups
    const int e = warp - 3;
    const int w = e >> 2;
    const int q4 = warp & 3;                 // TMEM lane quarter of this warp
    const unsigned lanes = (unsigned)(32 * q4) << 16;
    const int nloc = (nch - w + LGP_T4_NWG - 1) / LGP_T4_NWG;
    double* acc = accs + (size_t)w * LGP_TC_N * 128;  // [N][128] of this warpgroup
#pragma unroll
    for (int i = 0; i < LGP_TC_N; ++i) acc[i * 128 + 32 * q4 + lane] = 0.0;
    lgp_mbar_wait(TB4(T4B_AFULL), 0);
    const unsigned a1a = lgp_saddr(a1s);

    auto drain = [&](int gi) {
      const int b = gi & 1;
      lgp_mbar_wait(TB4(T4B_D2FULL(w, b)), (gi >> 1) & 1);
      lgp_tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        unsigned v[16];
        lgp_tmem_ld16(T4_D2(w, b) + lanes + 16u * h, v);
        lgp_tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i * 128 + 32 * q4 + lane] += (double)__uint_as_float(v[i]);
      }
      lgp_tc_fence_before();
      __syncwarp();
      if (lane == 0) lgp_mbar_arrive(TB4(T4B_D2EMPTY(w, b)));
    };

    for (int k = 0; k < nloc; ++k) {
      const int c = LGP_T4_NWG * k + w;
      const int st = c % LGP_TC_STAGES;
      lgp_mbar_wait(TB4(T4B_SFULL(st)), (c / LGP_TC_STAGES) & 1);  // column features staged
      const unsigned b1s = lgp_saddr(stg + (size_t)st * TC_STAGE_BYTES);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        // -r^2 of 16 rows x 64 columns, FP32 in registers
        float cf[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) cf[nt][i] = 0.f;
#pragma unroll
        for (int ks = 0; ks < LGP_TC_KD / 16; ++ks) {
          unsigned af[4];
          const int mi = lane >> 3;
          const int r = 32 * q4 + 16 * mt + (mi & 1) * 8 + (lane & 7);
          const int kc = 2 * ks + (mi >> 1);
          lgp_ldsm_x4(a1a + (unsigned)((r >> 3) * (LGP_TC_KD * 16) + kc * 128 + (r & 7) * 16), af);
#pragma unroll
          for (int nt = 0; nt < 8; ++nt) {
            const int nrow = 8 * nt + (lane & 7);
            const int kb = 2 * ks + ((lane >> 3) & 1);
            unsigned b0, b1;
            lgp_ldsm_x2(b1s + (unsigned)((nrow >> 3) * (LGP_TC_KD * 16) + kb * 128 + (nrow & 7) * 16),
                        b0, b1);
            lgp_hmma(cf[nt], af, b0, b1);
          }
        }
        unsigned hw[16], lw[16];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const int px = nt < (LGP_TC_POLY + 1) / 2 ? 1 : 0;
          const int px1 = nt < LGP_TC_POLY / 2 ? 1 : 0;
          float kv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) kv[i] = lgp_tc_k(LGP_TC_CLAMP(cf[nt][i]), a, (i & 1) ? px1 : px);
          lgp_split_f16x2(kv[0], kv[1], hw[2 * nt], lw[2 * nt]);
          lgp_split_f16x2(kv[2], kv[3], hw[2 * nt + 1], lw[2 * nt + 1]);
        }
        // P buffer of this warpgroup free once its previous contraction completed
        if (mt == 0 && k >= 1) lgp_mbar_wait(TB4(T4B_PEMPTY(w)), (k - 1) & 1);
        if (mt == 0) lgp_tc_fence_after();
        const unsigned pb = T4_P(w) + lanes + ((16u * mt) << 16);
        lgp_tmem_st16x128_x8(pb, hw);        // hi pairs: columns 0..31
        lgp_tmem_st16x128_x8(pb + 32u, lw);  // lo pairs: columns 32..63
      }
      lgp_tmem_wait_st();
      lgp_tc_fence_before();
      __syncwarp();
      if (lane == 0) lgp_mbar_arrive(TB4(T4B_PFULL(w)));
      if (k >= LGP_TC_DLAG && ((k - LGP_TC_DLAG) % LGP_TC_G) == LGP_TC_G - 1)
        drain((k - LGP_TC_DLAG) / LGP_TC_G);
    }
    for (int gi = nloc >= LGP_TC_DLAG ? (nloc - LGP_TC_DLAG) / LGP_TC_G : 0;
         gi < (nloc + LGP_TC_G - 1) / LGP_TC_G; ++gi)
      drain(gi);
    // combine the warpgroups' FP64 sums in a fixed order, undo the V scaling
    asm volatile("bar.sync 1, %0;" ::"r"(128 * LGP_T4_NWG) : "memory");
    if (w == 0) {
      const int row = 32 * q4 + lane;
      double* out = a.partial +
                    (((size_t)seg * a.n_pass + pass) * a.n_rows_pad + (size_t)rb * 128 + row) *
                        LGP_TC_N;
      const float* sc = a.vscale + (size_t)pass * LGP_TC_N;
#pragma unroll
      for (int i = 0; i < LGP_TC_N; i += 2) {
        double x0 = 0.0, x1 = 0.0;
#pragma unroll
        for (int u = 0; u < LGP_T4_NWG; ++u) {
          x0 += accs[((size_t)u * LGP_TC_N + i) * 128 + row];
          x1 += accs[((size_t)u * LGP_TC_N + i + 1) * 128 + row];
        }
        reinterpret_cast<double2*>(out)[i / 2] = make_double2(x0 * (double)sc[i], x1 * (double)sc[i + 1]);
      }
    }
  }
  lgp_tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    lgp_tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
#undef TB4
#undef T4_P
#undef T4_D2
}
#endif

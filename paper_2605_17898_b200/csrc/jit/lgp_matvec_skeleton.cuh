// JIT skeleton of the fused kernel-tree matvec (K1) and its FP64 companions.
//
// NVRTC compiles this text once per (kernel-tree structure, D, TB, tuning)
// after lgp_codegen.cpp has prepended:
//   - lgp_jit_abi.h                 (argument blocks)
//   - #define LGP_D / LGP_FR / LGP_FC / LGP_TB / LGP_R / LGP_THREADS / LGP_CC /
//             LGP_STAGES / LGP_SIGNED / LGP_MINB
//   - lgp_prep_point(), lgp_entry(), lgp_entry64()  (the compiled kernel tree)
//
// Replaces the reference slab loop (solvers.py:77-81: Kernel._gram on a row
// slab, then np.dot with v) without ever materialising a slab: kernel
// entries are generated in registers from per-point features and reduced
// against t right-hand sides in FP64.
//
// Data movement: column tiles of features (FP32) and packed RHS (FP64) are
// streamed HBM/L2 -> shared memory by the TMA bulk-copy engine
// (cp.async.bulk + mbarrier complete_tx), LGP_STAGES deep. Every thread of a
// CTA owns LGP_R rows (features in registers, LGP_R x LGP_TB FP64
// accumulators) and reads each column's features / RHS values from shared
// memory as warp-wide broadcasts.

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

// FP32 -> FP64 widening. Non-negative trees use an exact two-ALU-op bit
// construction (sign 0, exponent rebias +896, mantissa << 29) instead of
// F2F.F64.F32, which issues at 16/clk/SM on the same pipe class as MUFU.
// A zero input maps to 2^-127 (contributes < 1e-38 per entry).
__device__ __forceinline__ double lgp_widen(float f) {
#if LGP_SIGNED
  return (double)f;
#else
  const unsigned b = __float_as_uint(f);
  return __hiloint2double((b >> 3) + 0x38000000u, b << 29);
#endif
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
  while (!ok) {
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

#define LGP_ROWS_PER_CTA (LGP_THREADS * LGP_R)
#define LGP_FEAT_TILE_BYTES (LGP_CC * LGP_FC * 4)
#define LGP_V_TILE_BYTES (LGP_CC * LGP_TB * 8)
#define LGP_NWARPS (LGP_THREADS / 32)

// ---------------------------------------------------------------- features
extern "C" __global__ void lgp_prep(LgpPrepArgs p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_pad) return;
  float fr[LGP_FR];
  float fc[LGP_FC];
#pragma unroll
  for (int q = 0; q < LGP_FR; ++q) fr[q] = 0.f;
#pragma unroll
  for (int q = 0; q < LGP_FC; ++q) fc[q] = 0.f;
  if (i < p.n) {
    double x[LGP_D];
    const double* xp = p.x + (p.row0 + i) * LGP_D;
#pragma unroll
    for (int d = 0; d < LGP_D; ++d) x[d] = xp[d];
    lgp_prep_point(x, p, fr, fc);
  }
  if (p.fr) {
    float4* o = reinterpret_cast<float4*>(p.fr + i * LGP_FR);
#pragma unroll
    for (int q = 0; q < LGP_FR / 4; ++q)
      o[q] = make_float4(fr[4 * q], fr[4 * q + 1], fr[4 * q + 2], fr[4 * q + 3]);
  }
  if (p.fc) {
    float4* o = reinterpret_cast<float4*>(p.fc + i * LGP_FC);
#pragma unroll
    for (int q = 0; q < LGP_FC / 4; ++q)
      o[q] = make_float4(fc[4 * q], fc[4 * q + 1], fc[4 * q + 2], fc[4 * q + 3]);
  }
}

// ------------------------------------------------------------------- K1
extern "C" __global__ void __launch_bounds__(LGP_THREADS, LGP_MINB)
    lgp_matvec(const LgpMatvecArgs a) {
  if (a.done != nullptr && *a.done) return;
  const int item = blockIdx.x;
  const int rb = item % a.n_rb;
  const int rest = item / a.n_rb;
  const int seg = rest % a.n_seg;
  const int pass = rest / a.n_seg;
  const int tile0 = seg * a.tiles_per_seg;
  int ntiles = a.n_tiles - tile0;
  if (ntiles > a.tiles_per_seg) ntiles = a.tiles_per_seg;

  extern __shared__ __align__(128) unsigned char lgp_smem[];
  float* feat_s = reinterpret_cast<float*>(lgp_smem);
  double* v_s = reinterpret_cast<double*>(lgp_smem + LGP_STAGES * LGP_FEAT_TILE_BYTES);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(
      lgp_smem + LGP_STAGES * (LGP_FEAT_TILE_BYTES + LGP_V_TILE_BYTES));
  const unsigned full0 = lgp_saddr(bars);
  const unsigned empty0 = lgp_saddr(bars + LGP_STAGES);

  const int tid = threadIdx.x;
  const int lane = tid & 31;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < LGP_STAGES; ++s) {
      lgp_mbar_init(full0 + 8 * s, 1);
      lgp_mbar_init(empty0 + 8 * s, LGP_NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const float* fc_g = a.fc;
  const double* v_g = a.v + (size_t)pass * a.n_cols_pad * LGP_TB;
  auto issue = [&](int stage, int tile) {
    const unsigned bar = full0 + 8 * stage;
    lgp_mbar_expect_tx(bar, LGP_FEAT_TILE_BYTES + LGP_V_TILE_BYTES);
    lgp_bulk_g2s(lgp_saddr(feat_s + stage * (LGP_CC * LGP_FC)),
                 fc_g + (size_t)tile * LGP_CC * LGP_FC, LGP_FEAT_TILE_BYTES, bar);
    lgp_bulk_g2s(lgp_saddr(v_s + stage * (LGP_CC * LGP_TB)),
                 v_g + (size_t)tile * LGP_CC * LGP_TB, LGP_V_TILE_BYTES, bar);
  };
  if (tid == 0) {
    for (int s = 0; s < LGP_STAGES && s < ntiles; ++s) issue(s, tile0 + s);
  }

  // this thread's rows and their features (registers for the whole sweep)
  float fr[LGP_R][LGP_FR];
  const int row_base = rb * LGP_ROWS_PER_CTA + tid;
#pragma unroll
  for (int r = 0; r < LGP_R; ++r) {
    const float4* src =
        reinterpret_cast<const float4*>(a.fr + (size_t)(row_base + r * LGP_THREADS) * LGP_FR);
#pragma unroll
    for (int q = 0; q < LGP_FR / 4; ++q) {
      const float4 f4 = src[q];
      fr[r][4 * q] = f4.x;
      fr[r][4 * q + 1] = f4.y;
      fr[r][4 * q + 2] = f4.z;
      fr[r][4 * q + 3] = f4.w;
    }
  }

  double acc[LGP_R][LGP_TB];
#pragma unroll
  for (int r = 0; r < LGP_R; ++r)
#pragma unroll
    for (int c = 0; c < LGP_TB; ++c) acc[r][c] = 0.0;

  for (int it = 0; it < ntiles; ++it) {
    const int st = it % LGP_STAGES;
    const unsigned ph = (unsigned)(it / LGP_STAGES) & 1u;
    lgp_mbar_wait(full0 + 8 * st, ph);
    const float4* F = reinterpret_cast<const float4*>(feat_s + st * (LGP_CC * LGP_FC));
    const double* V = v_s + st * (LGP_CC * LGP_TB);
#pragma unroll 2
    for (int j = 0; j < LGP_CC; ++j) {
      float fc[LGP_FC];
#pragma unroll
      for (int q = 0; q < LGP_FC / 4; ++q) {
        const float4 f4 = F[j * (LGP_FC / 4) + q];
        fc[4 * q] = f4.x;
        fc[4 * q + 1] = f4.y;
        fc[4 * q + 2] = f4.z;
        fc[4 * q + 3] = f4.w;
      }
      double kd[LGP_R];
#pragma unroll
      for (int r = 0; r < LGP_R; ++r) kd[r] = lgp_widen(lgp_entry(fr[r], fc, a));
#if LGP_TB == 1
      const double vv = V[j];
#pragma unroll
      for (int r = 0; r < LGP_R; ++r) acc[r][0] = fma(kd[r], vv, acc[r][0]);
#else
      const double2* V2 = reinterpret_cast<const double2*>(V + j * LGP_TB);
#pragma unroll
      for (int c = 0; c < LGP_TB / 2; ++c) {
        const double2 vv = V2[c];
#pragma unroll
        for (int r = 0; r < LGP_R; ++r) {
          acc[r][2 * c] = fma(kd[r], vv.x, acc[r][2 * c]);
          acc[r][2 * c + 1] = fma(kd[r], vv.y, acc[r][2 * c + 1]);
        }
      }
#endif
    }
    __syncwarp();
    if (lane == 0) lgp_mbar_arrive(empty0 + 8 * st);
    if (tid == 0 && it + LGP_STAGES < ntiles) {
      lgp_mbar_wait(empty0 + 8 * st, ph);
      issue(st, tile0 + it + LGP_STAGES);
    }
  }

  double* out = a.partial + ((size_t)(seg * a.n_pass + pass) * a.n_rows_pad) * LGP_TB;
#pragma unroll
  for (int r = 0; r < LGP_R; ++r) {
    double* o = out + (size_t)(row_base + r * LGP_THREADS) * LGP_TB;
#if LGP_TB == 1
    o[0] = acc[r][0];
#else
#pragma unroll
    for (int c = 0; c < LGP_TB / 2; ++c)
      reinterpret_cast<double2*>(o)[c] = make_double2(acc[r][2 * c], acc[r][2 * c + 1]);
#endif
  }
}


// --------------------------------------------------- K1, symmetric operator
// K(X, X) is symmetric, so every off-diagonal block pair (I, J > I) is
// evaluated once and used twice: row side  out_I += K_IJ V_J  (registers) and
// column side out_J += K_IJ^T V_I (per-column warp reduction, then a fixed-
// order combine over warps). Diagonal blocks are evaluated in full, row side
// only. Halves the distance + transcendental work of the square operator;
// the FP32 entry k_ij is the same number on both sides, so the operator stays
// exactly symmetric. Partials are written per block pair and reduced in a
// fixed order by the epilogue (deterministic).
extern "C" __global__ void __launch_bounds__(LGP_THREADS, LGP_MINB)
    lgp_matvec_sym(const LgpMatvecArgs a) {
  if (a.done != nullptr && *a.done) return;
  const int unit = blockIdx.x;
  const int pass = blockIdx.y;
  const int I = a.units[2 * unit], J = a.units[2 * unit + 1];
  const bool offdiag = J != I;
  constexpr int TPB = LGP_ROWS_PER_CTA / LGP_CC;  // column tiles per block
  const int tile0 = J * TPB;
  const int ntiles = TPB;

  extern __shared__ __align__(128) unsigned char lgp_smem[];
  float* feat_s = reinterpret_cast<float*>(lgp_smem);
  double* v_s = reinterpret_cast<double*>(lgp_smem + LGP_STAGES * LGP_FEAT_TILE_BYTES);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(
      lgp_smem + LGP_STAGES * (LGP_FEAT_TILE_BYTES + LGP_V_TILE_BYTES));
  double* colbuf = reinterpret_cast<double*>(bars + 2 * LGP_STAGES);  // [NWARPS][CC][TB]
  const unsigned full0 = lgp_saddr(bars);
  const unsigned empty0 = lgp_saddr(bars + LGP_STAGES);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wid = tid >> 5;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < LGP_STAGES; ++s) {
      lgp_mbar_init(full0 + 8 * s, 1);
      lgp_mbar_init(empty0 + 8 * s, LGP_NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const double* v_g = a.v + (size_t)pass * a.n_cols_pad * LGP_TB;
  auto issue = [&](int stage, int tile) {
    const unsigned bar = full0 + 8 * stage;
    lgp_mbar_expect_tx(bar, LGP_FEAT_TILE_BYTES + LGP_V_TILE_BYTES);
    lgp_bulk_g2s(lgp_saddr(feat_s + stage * (LGP_CC * LGP_FC)),
                 a.fc + (size_t)tile * LGP_CC * LGP_FC, LGP_FEAT_TILE_BYTES, bar);
    lgp_bulk_g2s(lgp_saddr(v_s + stage * (LGP_CC * LGP_TB)),
                 v_g + (size_t)tile * LGP_CC * LGP_TB, LGP_V_TILE_BYTES, bar);
  };
  if (tid == 0) {
    for (int s = 0; s < LGP_STAGES && s < ntiles; ++s) issue(s, tile0 + s);
  }

  float fr[LGP_R][LGP_FR];
  double vr[LGP_R][LGP_TB];
  const int row_base = I * LGP_ROWS_PER_CTA + tid;
#pragma unroll
  for (int r = 0; r < LGP_R; ++r) {
    const int row = row_base + r * LGP_THREADS;
    const float4* src = reinterpret_cast<const float4*>(a.fr + (size_t)row * LGP_FR);
#pragma unroll
    for (int q = 0; q < LGP_FR / 4; ++q) {
      const float4 f4 = src[q];
      fr[r][4 * q] = f4.x;
      fr[r][4 * q + 1] = f4.y;
      fr[r][4 * q + 2] = f4.z;
      fr[r][4 * q + 3] = f4.w;
    }
#pragma unroll
    for (int c = 0; c < LGP_TB; ++c) vr[r][c] = v_g[(size_t)row * LGP_TB + c];
  }

  double acc[LGP_R][LGP_TB];
#pragma unroll
  for (int r = 0; r < LGP_R; ++r)
#pragma unroll
    for (int c = 0; c < LGP_TB; ++c) acc[r][c] = 0.0;

  double* colp = a.colpart + ((size_t)unit * gridDim.y + pass) * LGP_ROWS_PER_CTA * LGP_TB;
  for (int it = 0; it < ntiles; ++it) {
    const int st = it % LGP_STAGES;
    const unsigned ph = (unsigned)(it / LGP_STAGES) & 1u;
    lgp_mbar_wait(full0 + 8 * st, ph);
    const float4* F = reinterpret_cast<const float4*>(feat_s + st * (LGP_CC * LGP_FC));
    const double* V = v_s + st * (LGP_CC * LGP_TB);
#pragma unroll 2
    for (int j = 0; j < LGP_CC; ++j) {
      float fc[LGP_FC];
#pragma unroll
      for (int q = 0; q < LGP_FC / 4; ++q) {
        const float4 f4 = F[j * (LGP_FC / 4) + q];
        fc[4 * q] = f4.x;
        fc[4 * q + 1] = f4.y;
        fc[4 * q + 2] = f4.z;
        fc[4 * q + 3] = f4.w;
      }
      double vj[LGP_TB];
#pragma unroll
      for (int c = 0; c < LGP_TB; ++c) vj[c] = V[j * LGP_TB + c];
      double col[LGP_TB];
#pragma unroll
      for (int c = 0; c < LGP_TB; ++c) col[c] = 0.0;
#pragma unroll
      for (int r = 0; r < LGP_R; ++r) {
        const double kd = lgp_widen(lgp_entry(fr[r], fc, a));
#pragma unroll
        for (int c = 0; c < LGP_TB; ++c) {
          acc[r][c] = fma(kd, vj[c], acc[r][c]);
          col[c] = fma(kd, vr[r][c], col[c]);
        }
      }
      if (offdiag) {
#pragma unroll
        for (int c = 0; c < LGP_TB; ++c) {
          double v = col[c];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == (j & 31)) colbuf[(wid * LGP_CC + j) * LGP_TB + c] = v;
        }
      }
    }
    __syncwarp();
    if (lane == 0) lgp_mbar_arrive(empty0 + 8 * st);
    if (tid == 0 && it + LGP_STAGES < ntiles) {
      lgp_mbar_wait(empty0 + 8 * st, ph);
      issue(st, tile0 + it + LGP_STAGES);
    }
    if (offdiag) {
      __syncthreads();
      for (int e = tid; e < LGP_CC * LGP_TB; e += LGP_THREADS) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < LGP_NWARPS; ++w) s += colbuf[w * LGP_CC * LGP_TB + e];
        colp[(size_t)it * LGP_CC * LGP_TB + e] = s;
      }
      __syncthreads();
    }
  }

  double* out = a.partial + ((size_t)unit * gridDim.y + pass) * LGP_ROWS_PER_CTA * LGP_TB;
#pragma unroll
  for (int r = 0; r < LGP_R; ++r) {
    double* o = out + (size_t)(tid + r * LGP_THREADS) * LGP_TB;
#pragma unroll
    for (int c = 0; c < LGP_TB; ++c) o[c] = acc[r][c];
  }
}

// ------------------------------------------------------- FP64 companions
// Dense cross-covariance (kernel_eval) and diagonal (kernel_diag) in FP64,
// evaluated with direct differences: exactly symmetric for rows == cols.
extern "C" __global__ void lgp_gram(LgpGramArgs g) {
  const long long i = blockIdx.x;  // one row per CTA row-index (grid.x <= 2^31-1)
  double xi[LGP_D];
#pragma unroll
  for (int d = 0; d < LGP_D; ++d) xi[d] = g.x[i * LGP_D + d];
  for (long long j = (long long)blockIdx.y * blockDim.x + threadIdx.x; j < g.n_cols;
       j += (long long)gridDim.y * blockDim.x) {
    double xj[LGP_D];
#pragma unroll
    for (int d = 0; d < LGP_D; ++d) xj[d] = g.y[j * LGP_D + d];
    g.out[i * g.ld + j] = lgp_entry64(xi, xj, g);
  }
}

extern "C" __global__ void lgp_diag(LgpGramArgs g) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n_rows) return;
  double xi[LGP_D];
#pragma unroll
  for (int d = 0; d < LGP_D; ++d) xi[d] = g.x[i * LGP_D + d];
  g.out[i] = lgp_entry64(xi, xi, g);
}

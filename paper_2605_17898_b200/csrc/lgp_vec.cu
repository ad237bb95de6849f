// AOT (nvcc, sm_100a) FP64 vector kernels of the device-resident solver loops.
//
// All vectors are n x t row-major (the t right-hand sides / probes of one
// point contiguous). Column reductions are deterministic: a fixed
// (n, t) -> block partition, a fixed per-thread stride order, an in-order
// shared-memory combine, and a single-block in-order final sum. Scalar state
// (step sizes, residuals, activity masks) is written only by single-block
// "fin" kernels and read by the following launches, so no kernel races with
// itself. Every kernel returns immediately once the device `done` flag is
// set, which lets the host enqueue iterations ahead without syncing.
//
// Update formulas use explicit _rn intrinsics to keep the reference's
// rounding sequence (no FMA contraction): x += step*p, r -= step*ap,
// p = p*beta + r (solvers.py:115-121); w = w - a*q, w -= b*q_prev,
// w -= B^T (B w) (solvers.py:143-147).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "lgp_internal.h"

namespace lgp {
namespace vec {
namespace {

// fixed row partition of the deterministic reductions: enough blocks to keep
// every SM streaming (n = 100k -> 391 blocks of 256 rows)
constexpr int kMaxBlocks = 2048;
constexpr int kRowsPerBlock = 256;
// thread groups of the K1-TC-sym record epilogue (64 threads each)
constexpr int kTsGroups = 8;

inline int reduce_bd(int t) { return t * (256 / t); }

__device__ __forceinline__ bool is_done(const int* done) { return done != nullptr && *done; }

// sum of the records rec[e0 + g], rec[e0 + g + G], ... (< e1) at stride
// `width` doubles, column jj: 4 loads in flight per round, fixed order
template <int width>
__device__ __forceinline__ double sum_records(const double* __restrict__ data, const int* __restrict__ rec,
                                             int e0, int e1, int g, int jj) {
  double s = 0.0;
  int e = e0 + g;
  for (; e + 3 * kTsGroups < e1; e += 4 * kTsGroups) {
    int r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) r[u] = __ldg(rec + e + u * kTsGroups);
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = data[(size_t)r[u] * width + jj];
    s = (((s + v[0]) + v[1]) + v[2]) + v[3];
  }
  for (; e < e1; e += kTsGroups) s += data[(size_t)__ldg(rec + e) * width + jj];
  return s;
}


// sum_records for the column pair (jj, jj + 1) with 16-byte loads: the same
// records in the same order per column (bit-identical), up to 4 x 16 bytes in
// flight per round whatever the record count
template <int width>
__device__ __forceinline__ double2 sum_records2(const double* __restrict__ data, const int* __restrict__ rec,
                                                int e0, int e1, int g, int jj) {
  double sx = 0.0, sy = 0.0;
  for (int e = e0 + g; e < e1; e += 4 * kTsGroups) {
    int r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) r[u] = e + u * kTsGroups < e1 ? __ldg(rec + e + u * kTsGroups) : -1;
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      v[u] = r[u] >= 0 ? *reinterpret_cast<const double2*>(data + (size_t)r[u] * width + jj)
                       : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (r[u] >= 0) {
        sx += v[u].x;
        sy += v[u].y;
      }
  }
  return make_double2(sx, sy);
}

// block partial of sum_i a[i][c]*b[i][c] over this block's row range -> part[blk][c]
__device__ __forceinline__ void block_colsum(double v, int t, double* part_row, double* sm) {
  const int tid = threadIdx.x;
  const int bd = blockDim.x;
  sm[tid] = v;
  __syncthreads();
  if (tid < t) {
    double s = 0.0;
    for (int k = tid; k < bd; k += t) s += sm[k];
    part_row[tid] = s;
  }
  __syncthreads();
}

// Fixed-order (deterministic) column sums of part[nblk][t] by one block, for
// t <= blockDim.x / 2: thread (g, c) sums rows g, g + G, ... (G = power-of-two
// floor of blockDim.x / t), then a pairwise tree over g in shared memory.
// Afterwards sm[c] (c < t) holds column c's sum. All threads must call it.
// (A single thread per column walking all nblk rows was a ~400-long serial
// load + DADD chain: 18-25 us per CG / Lanczos scalar step at N = 100k.)
__device__ __forceinline__ bool part_par(int t) { return 2 * t <= 256; }
__device__ void part_colsums(const double* __restrict__ part, int nblk, int t, double* sm) {
  const int G = 1 << (31 - __clz((int)blockDim.x / t));
  const int tid = threadIdx.x, g = tid / t, c = tid - g * t;
  if (g < G) {
    double v = 0.0;
    for (int b = g; b < nblk; b += G) v += part[(size_t)b * t + c];
    sm[tid] = v;
  }
  __syncthreads();
  for (int h = G >> 1; h >= 1; h >>= 1) {
    if (g < h) sm[tid] += sm[tid + h * t];
    __syncthreads();
  }
}

// column c's sum: from sm after part_colsums when part_par(t), else serially
__device__ __forceinline__ double part_sum(const double* __restrict__ part, int nblk, int t, int c,
                                           const double* sm) {
  if (part_par(t)) return sm[c];
  double v = 0.0;
  for (int b = 0; b < nblk; ++b) v += part[(size_t)b * t + c];
  return v;
}

__global__ void k_dot_partial(const double* __restrict__ a, const double* __restrict__ b,
                              long long n, int t, long long chunk, double* part, const int* done) {
  __shared__ double sm[256];
  if (is_done(done)) return;
  const int tid = threadIdx.x;
  const int c = tid % t;
  const int stride = blockDim.x / t;
  const long long r0 = (long long)blockIdx.x * chunk;
  long long r1 = r0 + chunk;
  if (r1 > n) r1 = n;
  double s = 0.0;
  if (tid < stride * t)
    for (long long i = r0 + tid / t; i < r1; i += stride) s = fma(a[i * t + c], b[i * t + c], s);
  block_colsum(s, t, part + (size_t)blockIdx.x * t, sm);
}

__global__ void k_dot_final(const double* part, int nblk, int t, double* out, const int* done) {
  __shared__ double sm[256];
  if (is_done(done)) return;
  if (part_par(t)) part_colsums(part, nblk, t, sm);
  for (int c = threadIdx.x; c < t; c += blockDim.x) out[c] = part_sum(part, nblk, t, c, sm);
}

__global__ void k_pack(const double* __restrict__ V, long long n, int t, long long n_pad, int tb,
                       int n_pass, double* __restrict__ out, const int* done) {
  if (is_done(done)) return;
  const long long total = (long long)n_pass * n_pad * tb;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int cc = (int)(e % tb);
    const long long j = (e / tb) % n_pad;
    const int p = (int)(e / ((long long)tb * n_pad));
    const int c = p * tb + cc;
    double v = (j < n && c < t) ? V[j * t + c] : 0.0;
    out[e] = v;
  }
}

// power-of-two scale of each RHS column (max |V[:, c]| in [0.5, 1) after scaling)
// column max |V| (coalesced over the n x t block; order-free max through the
// bit patterns of non-negative doubles), then the power-of-two scales
__global__ void k_colmax(const double* __restrict__ V, long long n, int t,
                         unsigned long long* colmax, const int* done) {
  __shared__ double sm[256];
  if (is_done(done)) return;
  const int tid = threadIdx.x;
  const int c = tid % t;
  const int stride = blockDim.x / t;
  double m = 0.0;
  if (tid < stride * t)
    for (long long i = (long long)blockIdx.x * stride + tid / t; i < n;
         i += (long long)gridDim.x * stride)
      m = fmax(m, fabs(V[i * t + c]));
  sm[tid] = m;
  __syncthreads();
  if (tid < t) {
    double mm = 0.0;
    for (int k = tid; k < stride * t; k += t) mm = fmax(mm, sm[k]);
    if (mm > 0.0) atomicMax(colmax + tid, (unsigned long long)__double_as_longlong(mm));
  }
}

// t > 256: one thread per column (adjacent threads read adjacent columns)
__global__ void k_colmax_wide(const double* __restrict__ V, long long n, int t,
                              unsigned long long* colmax, const int* done) {
  if (is_done(done)) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= t) return;
  double m = 0.0;
  for (long long i = blockIdx.y; i < n; i += gridDim.y) m = fmax(m, fabs(V[i * t + c]));
  if (m > 0.0) atomicMax(colmax + c, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_colscale(const unsigned long long* __restrict__ colmax, int t, int ncols_pad,
                           float* scale, const int* done) {
  if (is_done(done)) return;
  for (int c = threadIdx.x; c < ncols_pad; c += blockDim.x) {
    double sc = 1.0;
    const double m = c < t ? __longlong_as_double((long long)colmax[c]) : 0.0;
    if (m > 0.0) {
      int e;
      frexp(m, &e);
      sc = ldexp(1.0, e);
    }
    scale[c] = (float)sc;
  }
}

// RHS tiles for the tensor-core K1: FP16 hi/lo of V / scale in the UMMA
// K-major canonical layout (rows = RHS c, K = column jj; 8-row groups of
// 8 x 128 B, 16-byte K chunks 128 B apart)
__global__ void k_pack_tc(const double* __restrict__ V, long long n, int t, int n_tiles, int tbn,
                          int n_pass, const float* __restrict__ scale, __half* __restrict__ out,
                          int* inexact, const int* done) {
  if (is_done(done)) return;
  const long long total = (long long)n_pass * n_tiles * tbn * 64;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int jj = (int)(e & 63);
    const int c = (int)((e >> 6) % tbn);
    const long long pt = (e >> 6) / tbn;  // pass * n_tiles + tile
    const long long tile = pt % n_tiles;
    const int pass = (int)(pt / n_tiles);
    const long long j = tile * 64 + jj;
    const int col = pass * tbn + c;
    const double v = (j < n && col < t) ? V[j * t + col] / (double)scale[col] : 0.0;
    const __half hi = __float2half_rn((float)v);
    const __half lo = __float2half_rn((float)(v - (double)__half2float(hi)));
    const int off = (c >> 3) * 512 + (jj >> 3) * 64 + (c & 7) * 8 + (jj & 7);
    __half* base = out + pt * 2 * tbn * 64;
    base[off] = hi;
    base[tbn * 64 + off] = lo;
    if (__half2float(lo) != 0.0f && *inexact == 0) atomicOr(inexact, 1);
  }
}

__global__ void k_epilogue(const double* __restrict__ partial, int n_seg, int n_pass,
                           long long rows_pad, int tb, long long n_rows, int t, double scale,
                           double noise, const double* __restrict__ noise_v,
                           double* __restrict__ out, const int* done) {
  if (is_done(done)) return;
  const long long total = n_rows * t;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / t;
    const int c = (int)(e % t);
    const int p = c / tb, cc = c % tb;
    double s = 0.0;
    for (int g = 0; g < n_seg; ++g) s += partial[(((long long)g * n_pass + p) * rows_pad + i) * tb + cc];
    double o = __dmul_rn(scale, s);
    if (noise_v != nullptr && noise != 0.0) o = __dadd_rn(o, __dmul_rn(noise, noise_v[e]));
    out[e] = o;
  }
}

__global__ void k_sym_epilogue(const double* __restrict__ rowp, const double* __restrict__ colp,
                               int nb, int rb, int n_pass, int tb, long long n, int t,
                               double scale, double noise, const double* __restrict__ noise_v,
                               double* __restrict__ out, const int* done) {
  if (is_done(done)) return;
  const long long total = n * t;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / t;
    const int c = (int)(e % t);
    const int p = c / tb, cc = c % tb;
    const int B = (int)(i / rb), il = (int)(i % rb);
    double s = 0.0;
    // row side of the block pairs (B, J >= B), then column side of (I < B, B)
    const long long uB = (long long)B * nb - (long long)B * (B - 1) / 2;
    for (int J = B; J < nb; ++J)
      s += rowp[(((uB + (J - B)) * n_pass + p) * rb + il) * tb + cc];
    for (int I = 0; I < B; ++I) {
      const long long u = (long long)I * nb - (long long)I * (I - 1) / 2 + (B - I);
      s += colp[((u * n_pass + p) * rb + il) * tb + cc];
    }
    double o = __dmul_rn(scale, s);
    if (noise_v != nullptr && noise != 0.0) o = __dadd_rn(o, __dmul_rn(noise, noise_v[e]));
    out[e] = o;
  }
}

__global__ void k_add_inplace(double* __restrict__ dst, const double* __restrict__ src, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = __dadd_rn(dst[i], src[i]);
}

__global__ void k_fill(double* p, long long n, double v) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    p[e] = v;
}

// ------------------------------------------------------------------ CG
__global__ void k_cg_init_vecs(const double* __restrict__ b, double* x, double* r, double* p,
                               long long total) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const double v = b[e];
    x[e] = 0.0;
    r[e] = v;
    p[e] = v;
  }
}

__global__ void k_cg_init_scalars(const double* bb, int t, double rel_tol, CgState s) {
  if (threadIdx.x == 0) {
    *s.status = 0;
    *s.bad_col = -1;
  }
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < t; c += blockDim.x) {
    const double bn = sqrt(bb[c]);
    s.tol[c] = rel_tol * bn;
    s.rs[c] = bb[c];
    s.step[c] = 0.0;
    s.beta[c] = 0.0;
    s.iters[c] = 0;
    s.res[c] = 0.0;
    const int act = bn != 0.0;  // zero column: 0 iterations, residual 0 (solvers.py:100-101)
    s.active[c] = act;
    if (act) atomicOr(&any, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) *s.done = any ? 0 : 1;
}

__global__ void k_cg_fin_pap(const double* part, int nblk, int t, CgState s) {
  __shared__ double sm[256];
  if (*s.done) return;
  if (part_par(t)) part_colsums(part, nblk, t, sm);
  for (int c = threadIdx.x; c < t; c += blockDim.x) {
    const double pap = part_sum(part, nblk, t, c, sm);
    if (s.active[c]) {
      if (pap <= 0.0) {  // breakdown: operator not SPD (solvers.py:110-113)
        *s.status = 1;
        *s.bad_col = c;
        *s.done = 1;
      }
      s.step[c] = s.rs[c] / pap;
    }
  }
}

__global__ void k_cg_update_xr(double* __restrict__ x, double* __restrict__ r,
                               const double* __restrict__ p, const double* __restrict__ ap,
                               long long n, int t, long long chunk, CgState s, double* part) {
  __shared__ double sm[256];
  if (*s.done) return;
  const int tid = threadIdx.x;
  const int c = tid % t;
  const int stride = blockDim.x / t;
  const long long r0 = (long long)blockIdx.x * chunk;
  long long r1 = r0 + chunk;
  if (r1 > n) r1 = n;
  double acc = 0.0;
  if (tid < stride * t) {
    const bool act = s.active[c] != 0;
    const double st = s.step[c];
    for (long long i = r0 + tid / t; i < r1; i += stride) {
      const long long e = i * t + c;
      double rv = r[e];
      if (act) {
        x[e] = __dadd_rn(x[e], __dmul_rn(st, p[e]));
        rv = __dsub_rn(rv, __dmul_rn(st, ap[e]));
        r[e] = rv;
      }
      acc = fma(rv, rv, acc);
    }
  }
  block_colsum(acc, t, part + (size_t)blockIdx.x * t, sm);
}

__global__ void k_cg_fin_rs(const double* part, int nblk, int t, int it, int max_iter,
                            CgState s) {
  __shared__ double sm[256];
  if (*s.done) return;
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  if (part_par(t)) part_colsums(part, nblk, t, sm);
  __syncthreads();
  for (int c = threadIdx.x; c < t; c += blockDim.x) {
    const double rs_new = part_sum(part, nblk, t, c, sm);
    if (!s.active[c]) continue;
    const double nrm = sqrt(rs_new);
    if (nrm <= s.tol[c] || it >= max_iter) {  // converged, or budget spent (reported)
      s.iters[c] = it;
      s.res[c] = nrm;
      s.active[c] = 0;
    } else {
      s.beta[c] = rs_new / s.rs[c];
      s.rs[c] = rs_new;
      atomicOr(&any, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && !any) *s.done = 1;
}

__global__ void k_cg_update_p(double* __restrict__ p, const double* __restrict__ r, long long total,
                              int t, CgState s) {
  if (*s.done) return;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % t);
    if (s.active[c]) p[e] = __dadd_rn(__dmul_rn(p[e], s.beta[c]), r[e]);
  }
}

// ------------------------------------------------- fused single-RHS CG
// The alpha solve (t = 1) runs 4 launches per iteration instead of 8:
//   pack   p = p * beta + r (update of the previous iteration) -> p, padded K1 operand
//   K1     (K1-TC-sym)
//   epi    row / column records -> Ap, its block's share of p.Ap, and in the
//          LAST block to finish: the fixed-order sum over blocks -> step,
//          breakdown check (solvers.py:108-113)
//   update x += step p, r -= step Ap, block shares of r.r, LAST block:
//          convergence / budget / beta (solvers.py:114-121)
// "Last block": each block writes its share, fences, takes a ticket; the
// block with the final ticket sums the shares in index order - the order
// never depends on which block finishes last (deterministic), and the scalar
// step needs no extra single-block launch.

// fixed-order sum of one value per thread over the block (any blockDim that
// is a multiple of 32): xor-shuffle tree per warp, then the warps in order
__device__ double block_sum_fixed(double v, double* sm) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += sm[w];
  return t;  // every thread holds the block sum
}

// block `blockIdx.x` deposits `val` (thread 0) into part[], returns true in
// the block that deposited last (which then sees every share)
__device__ bool deposit_last(double val, double* part, unsigned* counter, int nblk) {
  __shared__ unsigned ticket;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = val;
    __threadfence();
    ticket = atomicAdd(counter, 1u);
  }
  __syncthreads();
  const bool last = ticket == (unsigned)nblk - 1u;
  if (last) __threadfence();
  return last;
}

// fixed-order sum of part[0..nblk) by one block (the shares of other blocks
// are read through L2): threads 0..63 take every 64th share, whatever the
// block size, so kernels of different block sizes sum in the same order
__device__ double sum_shares(const double* part, int nblk, double* sm) {
  double v = 0.0;
  if (threadIdx.x < 64) {
    // 16 loads in flight per round (in-order issue would otherwise wait out
    // one L2 round trip per share); the adds keep the index order
    int b = threadIdx.x;
    for (; b + 15 * 64 < nblk; b += 16 * 64) {
      double x[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) x[u] = __ldcg(part + b + 64 * u);
#pragma unroll
      for (int u = 0; u < 16; ++u) v += x[u];
    }
    for (; b + 3 * 64 < nblk; b += 4 * 64) {
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = __ldcg(part + b + 64 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) v += x[u];
    }
    for (; b < nblk; b += 64) v += __ldcg(part + b);
  }
  return block_sum_fixed(v, sm);
}

__device__ void cg1_finish_pap(double pap, CgState s) {
  if (threadIdx.x == 0 && s.active[0]) {
    if (pap <= 0.0) {  // breakdown: operator not SPD (solvers.py:110-113)
      *s.status = 1;
      *s.bad_col = 0;
      *s.done = 1;
    }
    s.step[0] = s.rs[0] / pap;
  }
}

__global__ void k_cg1_pack(double* __restrict__ p, const double* __restrict__ r,
                           double* __restrict__ vpack, long long n, long long n_pad, CgState s) {
  if (*s.done) return;
  const double beta = s.beta[0];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad;
       i += (long long)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (i < n) {
      v = __dadd_rn(__dmul_rn(p[i], beta), r[i]);  // first iteration: beta = 0, p = r = b
      p[i] = v;
    }
    vpack[i] = v;
  }
}

// k_tcsym_epilogue + the p.Ap shares + the step (one RHS, one rank)
__global__ void __launch_bounds__(64 * kTsGroups)
    k_tcsym_epilogue_cg(const double* __restrict__ rowpart, const double* __restrict__ colpart,
                        const int* __restrict__ r_ptr, const int* __restrict__ r_rec,
                        const int* __restrict__ c_ptr, const int* __restrict__ c_rec, long long n,
                        double scale, double noise, const double* __restrict__ p,
                        double* __restrict__ out, double* part, unsigned* counter, CgState s) {
  __shared__ double pt[2][kTsGroups][64];
  __shared__ double sm[32];
  if (*s.done) return;
  const int c = blockIdx.x;
  const int jj = threadIdx.x & 63, g = threadIdx.x >> 6;
  const int I = c >> 1, r = (c & 1) * 64 + jj;
  pt[0][g][jj] = sum_records<64>(colpart, c_rec, c_ptr[c], c_ptr[c + 1], g, jj);
  pt[1][g][jj] = sum_records<128>(rowpart, r_rec, r_ptr[I], r_ptr[I + 1], g, r);
  __syncthreads();
  const long long i = (long long)c * 64 + jj;
  double d = 0.0;
  if (g == 0 && i < n) {
    double o = 0.0;
#pragma unroll
    for (int u = 0; u < kTsGroups; ++u) o += pt[0][u][jj];
#pragma unroll
    for (int u = 0; u < kTsGroups; ++u) o += pt[1][u][jj];
    o = __dmul_rn(scale, o);
    if (noise != 0.0) o = __dadd_rn(o, __dmul_rn(noise, p[i]));
    out[i] = o;
    d = p[i] * o;
  }
  const double share = block_sum_fixed(d, sm);
  if (deposit_last(share, part, counter, (int)gridDim.x)) {
    const double pap = sum_shares(part, (int)gridDim.x, sm);
    cg1_finish_pap(pap, s);
    if (threadIdx.x == 0) *counter = 0u;
  }
}

// p.Ap shares + the step (multi-rank CG, after the all-reduce of Ap): the
// same 64-row blocks and in-block order as k_tcsym_epilogue_cg, so a one-rank
// communicator reproduces the plain context bit for bit
__global__ void __launch_bounds__(64) k_cg1_pap(const double* __restrict__ p, const double* __restrict__ ap,
                                                long long n, double* part, unsigned* counter, CgState s) {
  __shared__ double sm[32];
  if (*s.done) return;
  const long long i = (long long)blockIdx.x * 64 + threadIdx.x;
  const double d = i < n ? p[i] * ap[i] : 0.0;
  const double share = block_sum_fixed(d, sm);
  if (deposit_last(share, part, counter, (int)gridDim.x)) {
    const double pap = sum_shares(part, (int)gridDim.x, sm);
    cg1_finish_pap(pap, s);
    if (threadIdx.x == 0) *counter = 0u;
  }
}

__global__ void __launch_bounds__(256) k_cg1_update(double* __restrict__ x, double* __restrict__ r,
                                                    const double* __restrict__ p,
                                                    const double* __restrict__ ap, long long n,
                                                    double* part, unsigned* counter, int it,
                                                    int max_iter, CgState s) {
  __shared__ double sm[32];
  if (*s.done) return;
  const double st = s.step[0];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(st, p[i]));
    const double rv = __dsub_rn(r[i], __dmul_rn(st, ap[i]));
    r[i] = rv;
    acc = fma(rv, rv, acc);
  }
  const double share = block_sum_fixed(acc, sm);
  if (deposit_last(share, part, counter, (int)gridDim.x)) {
    const double rs_new = sum_shares(part, (int)gridDim.x, sm);
    if (threadIdx.x == 0) {
      const double nrm = sqrt(rs_new);
      if (nrm <= s.tol[0] || it >= max_iter) {  // converged, or budget spent (reported)
        s.iters[0] = it;
        s.res[0] = nrm;
        s.active[0] = 0;
        *s.done = 1;
      } else {
        s.beta[0] = rs_new / s.rs[0];
        s.rs[0] = rs_new;
      }
      *counter = 0u;
    }
  }
}

// ------------------------------------------ one-launch CG vector step
// Everything of a single-RHS CG iteration except the matvec, as ONE
// cooperative launch (one CTA of 1024 threads per SM, co-resident): records
// -> Ap (+ noise p) and the p.Ap shares | grid barrier | step, x += step p,
// r -= step Ap and the r.r shares | grid barrier | beta / convergence, p =
// beta p + r and the K1 operand. Every CTA sums the shares itself (same fixed
// 64-lane order as sum_shares), so no CTA waits for a "last block", and the
// arithmetic is the 3-kernel sequence's bit for bit: the p.Ap shares are
// per 64-row block (k_tcsym_epilogue_cg / k_cg1_pap), the r.r shares per
// virtual 256-thread block of k_cg1_update's grid-stride layout. With
// rowpart == nullptr the records phase is skipped and Ap is read as given
// (the multi-rank CG, after its all-reduce).
constexpr int kVecThreads = 1024;
constexpr int kVecQB = kVecThreads / 256;  // 64-row blocks per record round

// generation barrier over the co-resident grid: bar[0] arrivals, bar[1]
// generation (a flag per CTA polled by every CTA measured 10 us, this 2 us)
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1u) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// sum_shares with the shares staged through shared memory by the whole CTA
// (one L2 round trip for up to `cap` shares instead of one per 16 per lane):
// lane L still adds the shares b = L (mod 64) in index order (cap % 64 == 0)
__device__ double sum_shares_staged(const double* part, int nblk, double* stg, int cap, double* sm) {
  double v = 0.0;
  for (int base = 0; base < nblk; base += cap) {
    const int m = min(cap, nblk - base);
    for (int k = threadIdx.x; k < m; k += blockDim.x) stg[k] = __ldcg(part + base + k);
    __syncthreads();
    if (threadIdx.x < 64)
      for (int k = threadIdx.x; k < m; k += 64) v += stg[k];
    __syncthreads();
  }
  return block_sum_fixed(v, sm);
}

__global__ void __launch_bounds__(kVecThreads, 1)
    k_cg1_vec(const double* __restrict__ rowpart, const double* __restrict__ colpart,
              const int* __restrict__ r_ptr, const int* __restrict__ r_rec, const int* __restrict__ c_ptr,
              const int* __restrict__ c_rec, long long n, long long n_pad, double scale, double noise,
              double* x, double* r, double* p, double* ap, double* vpack, double* part_pap,
              double* part_rs, int nvb, unsigned* bar, int it, int max_iter, CgState s,
              unsigned long long* trace) {
  // trace (diagnostics, LGP_CG_VEC_TRACE): %globaltimer at the phase
  // boundaries, per CTA
  auto stamp = [&](int k) {
    if (trace != nullptr && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[(size_t)blockIdx.x * 8 + k] = t;
    }
  };
  stamp(0);
  __shared__ double pt[kVecQB][2][kTsGroups][64];
  __shared__ double sm[32];
  __shared__ double ws[32];
  if (*s.done) return;  // written only by earlier launches: the same for every CTA
  const double rs_old = s.rs[0];
  const long long nc = (n + 63) / 64;
  {
    // ---- records -> Ap, p.Ap share of each 64-row block: kVecQB blocks per
    // round, 256 threads each = 8 record groups x 32 column pairs (measured:
    // 128 threads x 4 columns 10.1 us, both lists' loads interleaved 9.1 us,
    // this 8.6 us at cfg4: the record reads are throughput-, not latency-bound)
    const int qb = threadIdx.x >> 8, lt = threadIdx.x & 255;
    const int j2 = 2 * (lt & 31), g = lt >> 5;
    // record-list bounds of this thread's block, one round ahead (the
    // bounds -> indices -> records chain is three dependent L2 round trips)
    auto bounds = [&](long long c, int4& e) {
      if (c < nc) {
        const int I = (int)(c >> 1);
        e = make_int4(__ldg(c_ptr + c), __ldg(c_ptr + c + 1), __ldg(r_ptr + I), __ldg(r_ptr + I + 1));
      }
    };
    const bool recs = rowpart != nullptr;  // else Ap is given (multi-rank: all-reduced)
    int4 eb = make_int4(0, 0, 0, 0), en = eb;
    if (recs) bounds((long long)kVecQB * blockIdx.x + qb, eb);
    for (long long c0 = (long long)kVecQB * blockIdx.x; c0 < nc; c0 += (long long)kVecQB * gridDim.x) {
      const long long c = c0 + qb;
      if (recs) bounds(c + (long long)kVecQB * gridDim.x, en);
      // this block's p entries, loaded alongside the records
      const double pi = (lt < 64 && c < nc && c * 64 + lt < n) ? p[c * 64 + lt] : 0.0;
      if (recs && c < nc) {
        const int rr = (int)(c & 1) * 64 + j2;
        const double2 cs = sum_records2<64>(colpart, c_rec, eb.x, eb.y, g, j2);
        const double2 rs = sum_records2<128>(rowpart, r_rec, eb.z, eb.w, g, rr);
        pt[qb][0][g][j2] = cs.x;
        pt[qb][0][g][j2 + 1] = cs.y;
        pt[qb][1][g][j2] = rs.x;
        pt[qb][1][g][j2 + 1] = rs.y;
      }
      __syncthreads();
      if (lt < 64) {
        const int jj = lt;
        const long long i = c * 64 + jj;
        double d = 0.0;
        if (c < nc && i < n) {
          if (recs) {
            double o = 0.0;
#pragma unroll
            for (int u = 0; u < kTsGroups; ++u) o += pt[qb][0][u][jj];
#pragma unroll
            for (int u = 0; u < kTsGroups; ++u) o += pt[qb][1][u][jj];
            o = __dmul_rn(scale, o);
            if (noise != 0.0) o = __dadd_rn(o, __dmul_rn(noise, pi));
            ap[i] = o;
            d = pi * o;
          } else {
            d = pi * ap[i];  // k_cg1_pap's share
          }
        }
        // block_sum_fixed of the 64-thread block: each warp's xor tree, then
        // the two warps in order
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if ((lt & 31) == 0) ws[2 * qb + (lt >> 5)] = d;
      }
      __syncthreads();
      if (c < nc && lt == 0) part_pap[c] = (0.0 + ws[2 * qb]) + ws[2 * qb + 1];
      eb = en;
    }
  }
  stamp(1);
  grid_sync(bar);
  stamp(2);
  double* stg = &pt[0][0][0][0];  // the record buffers are free now
  const double pap = sum_shares_staged(part_pap, (int)nc, stg, kVecQB * 2 * kTsGroups * 64, sm);
  stamp(3);
  const double st = rs_old / pap;
  if (pap <= 0.0) {  // breakdown: operator not SPD (solvers.py:110-113)
    if (blockIdx.x == 0 && threadIdx.x == 0 && s.active[0]) {
      *s.status = 1;
      *s.bad_col = 0;
      *s.done = 1;
      s.step[0] = st;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) s.step[0] = st;
  // ---- x, r update and the r.r share of each virtual block (k_cg1_update)
  const int vb = blockIdx.x * (kVecThreads / 256) + (threadIdx.x >> 8);
  const long long stride = (long long)nvb * 256;
  double acc = 0.0;
  if (vb < nvb) {
    for (long long i = (long long)vb * 256 + (threadIdx.x & 255); i < n; i += stride) {
      x[i] = __dadd_rn(x[i], __dmul_rn(st, p[i]));
      const double rv = __dsub_rn(r[i], __dmul_rn(st, __ldcg(ap + i)));  // ap: other CTAs' stores
      r[i] = rv;
      acc = fma(rv, rv, acc);
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __syncthreads();  // ws reuse
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (vb < nvb && (threadIdx.x & 255) == 0) {
    double t = 0.0;
    const int w0 = threadIdx.x >> 5;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += ws[w0 + w];
    part_rs[vb] = t;
  }
  stamp(4);
  grid_sync(bar);
  stamp(5);
  const double rs_new = sum_shares_staged(part_rs, nvb, stg, kVecQB * 2 * kTsGroups * 64, sm);
  stamp(6);
  const double nrm = sqrt(rs_new);
  if (nrm <= s.tol[0] || it >= max_iter) {  // converged, or budget spent (reported)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      s.iters[0] = it;
      s.res[0] = nrm;
      s.active[0] = 0;
      *s.done = 1;
    }
    return;
  }
  const double beta = rs_new / rs_old;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s.beta[0] = beta;
    s.rs[0] = rs_new;
  }
  // ---- p = beta p + r (the next iteration's direction) and the K1 operand
  if (vb < nvb) {
    for (long long i = (long long)vb * 256 + (threadIdx.x & 255); i < n; i += stride) {
      const double v = __dadd_rn(__dmul_rn(p[i], beta), r[i]);
      p[i] = v;
      vpack[i] = v;
    }
  }
  stamp(7);
}

// ------------------------------------------------ multi-shift CG (CG-M)
// (K + (noise + sig_e) I) x_e = b for all e at one matvec per iteration:
// the shifted systems' residuals stay collinear with the seed's,
// r_e = zeta_e r, so each needs only its own scalars and two vectors
// (Jegerlehner 1996). With the seed's CG coefficients alpha_k, beta_k:
//   zeta_{k+1} = zeta_k zeta_{k-1} a_{k-1} /
//                (zeta_{k-1} a_{k-1} (1 + a_k sig) + a_k b_{k-1} (zeta_{k-1} - zeta_k))
//   a^e_k = a_k zeta_{k+1} / zeta_k,   b^e_k = b_k (zeta_{k+1} / zeta_k)^2
//   x^e += a^e_k p^e;   p^e = zeta_{k+1} r_{k+1} + b^e_k p^e
// stop when |zeta_{k+1}| ||r_{k+1}|| <= tol ||b|| (the shifted system's own
// recurrence residual: the reference's per-solve rule, solvers.py:114-119).
// State double-buffered by iteration parity (every block reads [it & 1],
// block 0 writes [(it + 1) & 1]).
__global__ void k_cg_shift_init(const double* __restrict__ b, long long n, int nsh,
                                double* __restrict__ xs, double* __restrict__ ps, CgShiftState* st) {
  const long long total = n * nsh;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    xs[e] = 0.0;
    ps[e] = b[e / nsh];
  }
  if (blockIdx.x == 0) {
    CgShiftState* c = st + 1;  // the state the first iteration (it = 1) reads
    for (int e = threadIdx.x; e < nsh; e += blockDim.x) {
      c->z[e] = 1.0;
      c->zm1[e] = 1.0;
      c->active[e] = 1;
      c->iters[e] = 0;
      c->res[e] = 0.0;
    }
    if (threadIdx.x == 0) {
      c->am1 = 1.0;
      c->bm1 = 0.0;
    }
  }
}

__global__ void __launch_bounds__(256) k_cg_shift(double* __restrict__ xs, double* __restrict__ ps,
                                                  const double* __restrict__ r, long long n, int nsh,
                                                  const double* __restrict__ sig, CgShiftState* st,
                                                  CgState s, int it) {
  __shared__ double sa[kMaxShifts], sb[kMaxShifts], sz[kMaxShifts];
  __shared__ int sact[kMaxShifts];
  // the seed finished at an earlier iteration: nothing left to apply
  if (*s.done && s.iters[0] != it) return;
  const bool seed_done = *s.done != 0;  // (then s.iters[0] == it: its last iteration)
  const CgShiftState* cur = st + (it & 1);
  CgShiftState* nxt = st + ((it + 1) & 1);
  const double ak = s.step[0];
  const double bk = seed_done ? 0.0 : s.beta[0];
  const double nrm = seed_done ? s.res[0] : sqrt(s.rs[0]);  // ||r_{k+1}|| of the seed
  for (int e = threadIdx.x; e < nsh; e += blockDim.x) {
    const int act = cur->active[e];
    const double zk = cur->z[e], zkm1 = cur->zm1[e];
    double zn = zk, a = 0.0, be = 0.0;
    if (act) {
      const double den = zkm1 * cur->am1 * (1.0 + ak * sig[e]) + ak * cur->bm1 * (zkm1 - zk);
      zn = zk * zkm1 * cur->am1 / den;
      a = ak * (zn / zk);
      be = bk * ((zn / zk) * (zn / zk));
    }
    sa[e] = a;
    sb[e] = be;
    sz[e] = zn;
    sact[e] = act;
    if (blockIdx.x == 0) {
      nxt->z[e] = zn;
      nxt->zm1[e] = zk;
      int a2 = act, iters = cur->iters[e];
      double res = cur->res[e];
      if (act) {
        const double rn = fabs(zn) * nrm;
        if (rn <= s.tol[0] || seed_done) {  // converged, or the seed (slowest) stopped
          a2 = 0;
          iters = it;
          res = rn;
        }
      }
      nxt->active[e] = a2;
      nxt->iters[e] = iters;
      nxt->res[e] = res;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    nxt->am1 = ak;
    nxt->bm1 = bk;
  }
  __syncthreads();
  const long long total = n * nsh;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(q % nsh);
    if (!sact[e]) continue;
    const double pv = ps[q];
    xs[q] = __dadd_rn(xs[q], __dmul_rn(sa[e], pv));
    ps[q] = __dadd_rn(__dmul_rn(pv, sb[e]), __dmul_rn(sz[e], r[q / nsh]));
  }
}

// --------------------------------------- column compaction (multi-RHS CG)
// dst[i][k] = src[i][map[k]] (k < t_run) and back: the multi-RHS CG runs its
// K1 passes on the still-active columns only
__global__ void k_gather_cols(const double* __restrict__ src, long long n, int t,
                              const int* __restrict__ map, int t_run, double* __restrict__ dst,
                              const int* done) {
  if (is_done(done)) return;
  const long long total = n * t_run;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / t_run;
    const int k = (int)(e - i * t_run);
    dst[e] = src[i * t + map[k]];
  }
}

__global__ void k_scatter_cols(const double* __restrict__ src, long long n, int t_run,
                               const int* __restrict__ map, int t, double* __restrict__ dst,
                               const int* done) {
  if (is_done(done)) return;
  const long long total = n * t_run;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / t_run;
    const int k = (int)(e - i * t_run);
    dst[i * t + map[k]] = src[e];
  }
}

// ------------------------------------------------------------- Lanczos
__global__ void k_lz_init(const double* __restrict__ z, double* __restrict__ q, long long total,
                          int t, const double* zz) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % t);
    q[e] = z[e] / sqrt(zz[c]);
  }
}

__global__ void k_lz_init_scalars(const double* zz, int t, LzState s) {
  for (int c = threadIdx.x; c < t; c += blockDim.x) {
    s.active[c] = zz[c] > 0.0;
    s.count[c] = 0;
  }
  if (threadIdx.x == 0) *s.done = 0;
}

__global__ void k_lz_fin_alpha(const double* part, int nblk, int t, int j, int steps, LzState s) {
  __shared__ double sm[256];
  if (*s.done) return;
  if (part_par(t)) part_colsums(part, nblk, t, sm);
  for (int c = threadIdx.x; c < t; c += blockDim.x) {
    const double a = part_sum(part, nblk, t, c, sm);
    if (s.active[c]) {
      s.alpha[(size_t)c * steps + j] = a;
      s.a_cur[c] = a;
      s.count[c] = j + 1;
    }
  }
}

__global__ void k_lz_update1(double* __restrict__ w, const double* __restrict__ q,
                             const double* __restrict__ qprev, long long total, int t, int j,
                             int steps, LzState s) {
  if (*s.done) return;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % t);
    if (!s.active[c]) {
      w[e] = 0.0;
      continue;
    }
    double v = __dsub_rn(w[e], __dmul_rn(s.a_cur[c], q[e]));
    if (j > 0) v = __dsub_rn(v, __dmul_rn(s.beta[(size_t)c * steps + j - 1], qprev[e]));
    w[e] = v;
  }
}

// part[blk][k][c] = sum over this block's rows of basis[k][i][c] * w[i][c], k < nb
constexpr int kLzBatch = 8;
__global__ void k_lz_multidot(const double* __restrict__ basis, long long stride_k, int nb,
                              const double* __restrict__ w, long long n, int t, long long chunk,
                              double* part, const int* done) {
  __shared__ double sm[kLzBatch * 256];
  if (is_done(done)) return;
  const int tid = threadIdx.x;
  const int bd = blockDim.x;  // = t * (256 / t): every thread owns a column
  const int c = tid % t;
  const int stride = bd / t;
  const long long r0 = (long long)blockIdx.x * chunk;
  long long r1 = r0 + chunk;
  if (r1 > n) r1 = n;
  // basis vectors in batches of 8: w is read once per batch, 8 independent
  // FMA chains keep loads in flight, and one shared-memory pass reduces the
  // batch (per-(k, c) summation order: rows in stride order, then the block's
  // threads of column c in tid order, as block_colsum)
  for (int k0 = 0; k0 < nb; k0 += kLzBatch) {
    double s[kLzBatch];
#pragma unroll
    for (int kk = 0; kk < kLzBatch; ++kk) s[kk] = 0.0;
    // 4 rows per iteration: all 4 x (1 + 8) loads issue before the FMAs
    // (one memory latency per 4 rows instead of per row)
    long long i = r0 + tid / t;
    for (; i + 3 * stride < r1; i += 4 * stride) {
      double wv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) wv[u] = w[(i + u * stride) * t + c];
#pragma unroll
      for (int kk = 0; kk < kLzBatch; ++kk)
        if (k0 + kk < nb) {
          const double* bk = basis + (size_t)(k0 + kk) * stride_k + c;
          double bv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) bv[u] = bk[(i + u * stride) * t];
#pragma unroll
          for (int u = 0; u < 4; ++u) s[kk] = fma(bv[u], wv[u], s[kk]);
        }
    }
    for (; i < r1; i += stride) {
      const long long e = i * t + c;
      const double wv = w[e];
#pragma unroll
      for (int kk = 0; kk < kLzBatch; ++kk)
        if (k0 + kk < nb) s[kk] = fma(basis[(size_t)(k0 + kk) * stride_k + e], wv, s[kk]);
    }
#pragma unroll
    for (int kk = 0; kk < kLzBatch; ++kk) sm[kk * 256 + tid] = s[kk];
    __syncthreads();
    for (int o = tid; o < kLzBatch * t; o += bd) {
      const int kk = o / t, cc = o - kk * t;
      if (k0 + kk < nb) {
        double r = 0.0;
        for (int q = cc; q < bd; q += t) r += sm[kk * 256 + q];
        part[((size_t)blockIdx.x * nb + k0 + kk) * t + cc] = r;
      }
    }
    __syncthreads();
  }
}

// Same partials, one (k, c) pair per thread: block (row chunk, k group of
// blockDim / t basis vectors); no shared-memory reduction, 8 rows in flight.
// part[blk][k][c] = sum over the chunk's rows, in row order.
__global__ void __launch_bounds__(256) k_lz_multidot2(const double* __restrict__ basis,
                                                      long long stride_k, int nb,
                                                      const double* __restrict__ w, long long n,
                                                      int t, long long chunk, double* part,
                                                      const int* done) {
  if (is_done(done)) return;
  const int kb = blockDim.x / t;
  const int kk = threadIdx.x / t, c = threadIdx.x - kk * t;
  const int k = blockIdx.y * kb + kk;
  if (kk >= kb || k >= nb) return;
  const long long r0 = (long long)blockIdx.x * chunk;
  long long r1 = r0 + chunk;
  if (r1 > n) r1 = n;
  const double* __restrict__ bk = basis + (size_t)k * stride_k + c;
  const double* __restrict__ wc = w + c;
  double s = 0.0;
  long long i = r0;
  for (; i + 8 <= r1; i += 8) {
    double bv[8], wv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      bv[u] = bk[(i + u) * t];
      wv[u] = wc[(i + u) * t];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) s = fma(bv[u], wv[u], s);
  }
  for (; i < r1; ++i) s = fma(bk[i * t], wc[i * t], s);
  part[((size_t)blockIdx.x * nb + k) * t + c] = s;
}

// h[e] = sum over blocks of part[blk][e], e < m = nb * t: 32 entries per block
// (coalesced rows), 8 warps over the blocks (b = warp, warp + 8, ...), combined
// in warp order (deterministic)
__global__ void __launch_bounds__(256) k_lz_fin_h(const double* part, int nblk, int nb, int t,
                                                  LzState s) {
  __shared__ double sm[8][32];
  if (*s.done) return;
  const int m = nb * t;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  double v = 0.0;
  if (e < m)
    for (int b = wp; b < nblk; b += 8) v += part[(size_t)b * m + e];
  sm[wp][lane] = v;
  __syncthreads();
  if (wp == 0 && e < m) {
    double h = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) h += sm[u][lane];
    s.h[e] = h;
  }
}

__global__ void k_lz_update2(double* __restrict__ w, const double* __restrict__ basis,
                             long long stride_k, int nb, long long n, int t, long long chunk,
                             LzState s, double* part) {
  __shared__ double sm[256];
  __shared__ double hs[64 * 32];  // h[k][c] for nb <= 64, t <= 32 (else read from global)
  if (*s.done) return;
  const int tid = threadIdx.x;
  const int c = tid % t;
  const int stride = blockDim.x / t;
  const long long r0 = (long long)blockIdx.x * chunk;
  long long r1 = r0 + chunk;
  if (r1 > n) r1 = n;
  const bool hsm = nb * t <= 64 * 32;
  if (hsm)
    for (int e = tid; e < nb * t; e += blockDim.x) hs[e] = s.h[e];
  __syncthreads();
  const double* h = hsm ? hs : s.h;
  double acc = 0.0;
  if (tid < stride * t) {
    const bool act = s.active[c] != 0;
    // two rows per iteration, 8 independent chains over k each (16 loads in
    // flight), summed pairwise; per-row arithmetic identical for both loops
    long long i = r0 + tid / t;
    for (; i + stride < r1; i += 2 * stride) {
      const long long e0 = i * t + c, e1 = e0 + (long long)stride * t;
      double v0 = w[e0], v1 = w[e1];
      if (act) {
        double a8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        double b8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        int k = 0;
        for (; k + 8 <= nb; k += 8) {
          double x0[8], x1[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            x0[kk] = basis[(size_t)(k + kk) * stride_k + e0];
            x1[kk] = basis[(size_t)(k + kk) * stride_k + e1];
          }
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const double hk = h[(k + kk) * t + c];
            a8[kk] = fma(x0[kk], hk, a8[kk]);
            b8[kk] = fma(x1[kk], hk, b8[kk]);
          }
        }
        for (; k < nb; ++k) {
          const double hk = h[k * t + c];
          a8[0] = fma(basis[(size_t)k * stride_k + e0], hk, a8[0]);
          b8[0] = fma(basis[(size_t)k * stride_k + e1], hk, b8[0]);
        }
        const double u0 = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
        const double u1 = ((b8[0] + b8[1]) + (b8[2] + b8[3])) + ((b8[4] + b8[5]) + (b8[6] + b8[7]));
        v0 = __dsub_rn(v0, u0);
        v1 = __dsub_rn(v1, u1);
        w[e0] = v0;
        w[e1] = v1;
      }
      acc = fma(v0, v0, acc);
      acc = fma(v1, v1, acc);
    }
    for (; i < r1; i += stride) {
      const long long e = i * t + c;
      double v = w[e];
      if (act) {
        double u8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        int k = 0;
        for (; k + 8 <= nb; k += 8)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            u8[kk] = fma(basis[(size_t)(k + kk) * stride_k + e], h[(k + kk) * t + c], u8[kk]);
        for (; k < nb; ++k) u8[0] = fma(basis[(size_t)k * stride_k + e], h[k * t + c], u8[0]);
        const double u = ((u8[0] + u8[1]) + (u8[2] + u8[3])) + ((u8[4] + u8[5]) + (u8[6] + u8[7]));
        v = __dsub_rn(v, u);
        w[e] = v;
      }
      acc = fma(v, v, acc);
    }
  }
  block_colsum(acc, t, part + (size_t)blockIdx.x * t, sm);
}

__global__ void k_lz_fin_beta(const double* part, int nblk, int t, int j, int steps, LzState s) {
  __shared__ double sm[256];
  if (*s.done) return;
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  if (part_par(t)) part_colsums(part, nblk, t, sm);
  __syncthreads();
  for (int c = threadIdx.x; c < t; c += blockDim.x) {
    const double ss = part_sum(part, nblk, t, c, sm);
    if (!s.active[c]) continue;
    const double nb = sqrt(ss);
    const double a = fabs(s.a_cur[c]);
    if (nb <= 1e-12 * (a > 1.0 ? a : 1.0)) {  // invariant subspace (solvers.py:151-152)
      s.active[c] = 0;
    } else {
      s.beta[(size_t)c * steps + j] = nb;
      s.nrm[c] = nb;
      atomicOr(&any, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && !any) *s.done = 1;
}

__global__ void k_lz_normalize(const double* __restrict__ w, double* __restrict__ q,
                               long long total, int t, LzState s) {
  if (*s.done) return;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % t);
    q[e] = s.active[c] ? w[e] / s.nrm[c] : 0.0;
  }
}

// ---- point-set statistics (lgp_points_upload): column means, finiteness,
// radius about the mean. Block (b, j) sums column j over row chunk b in a
// fixed order, so the mean is deterministic (and identical on every rank).
__global__ void k_pt_colsum(const double* __restrict__ x, long long n, int d, long long rows,
                            double* __restrict__ part, int* bad) {
  const int j = blockIdx.y;
  const long long r0 = (long long)blockIdx.x * rows;
  long long r1 = r0 + rows;
  if (r1 > n) r1 = n;
  double acc = 0.0;
  int nf = 0;
  for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const double v = x[i * d + j];
    nf |= !isfinite(v);
    acc += v;
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(long long)blockIdx.x * d + j] = sh[0];
  if (nf) atomicOr(bad, 1);
}

// one warp per column: lane-strided partial sums, then a fixed butterfly
// (deterministic order)
__global__ void k_pt_center(const double* __restrict__ part, int nblk, int d, long long n,
                            double* ctr, double* stats) {
  const int lane = threadIdx.x & 31;
  for (int j = threadIdx.x >> 5; j < d; j += blockDim.x >> 5) {
    double acc = 0.0;
    for (int b = lane; b < nblk; b += 32) acc += part[(long long)b * d + j];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const double c = n > 0 ? acc / (double)n : 0.0;
      ctr[j] = c;
      stats[j] = c;
    }
  }
}

__global__ void k_pt_radius(const double* __restrict__ x, long long n, int d,
                            const double* __restrict__ ctr, unsigned long long* r2max) {
  double m = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double r2 = 0.0;
    for (int j = 0; j < d; ++j) {
      const double e = x[i * d + j] - ctr[j];
      r2 += e * e;
    }
    m = fmax(m, r2);
  }
  // non-negative doubles order like their bit patterns
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && isfinite(m)) atomicMax(r2max, __double_as_longlong(m));
}

// One block per 64-column chunk c: out[64c + jj] = scale * (the column
// records of chunk c + the row records of row block I = c / 2) + noise * v.
// Each side's sum is split over kTsGroups thread groups (group g takes list
// entries g, g + G, ...) and combined in g order, column side first: fixed
// order, deterministic.
__global__ void __launch_bounds__(64 * kTsGroups)
    k_tcsym_epilogue(const double* __restrict__ rowpart, const double* __restrict__ colpart,
                     const int* __restrict__ r_ptr, const int* __restrict__ r_rec,
                     const int* __restrict__ c_ptr, const int* __restrict__ c_rec, long long n,
                     double scale, double noise, const double* __restrict__ noise_v,
                     double* __restrict__ out, const int* done) {
  __shared__ double part[2][kTsGroups][64];
  if (is_done(done)) return;
  const int c = blockIdx.x;
  const int jj = threadIdx.x & 63, g = threadIdx.x >> 6;
  const int I = c >> 1, r = (c & 1) * 64 + jj;
  part[0][g][jj] = sum_records<64>(colpart, c_rec, c_ptr[c], c_ptr[c + 1], g, jj);
  part[1][g][jj] = sum_records<128>(rowpart, r_rec, r_ptr[I], r_ptr[I + 1], g, r);
  __syncthreads();
  const long long i = (long long)c * 64 + jj;
  if (g == 0 && i < n) {
    double o = 0.0;
#pragma unroll
    for (int u = 0; u < kTsGroups; ++u) o += part[0][u][jj];
#pragma unroll
    for (int u = 0; u < kTsGroups; ++u) o += part[1][u][jj];
    o = __dmul_rn(scale, o);
    if (noise_v != nullptr && noise != 0.0) o = __dadd_rn(o, __dmul_rn(noise, noise_v[i]));
    out[i] = o;
  }
}

inline int grid_for(long long total, int bd = 256) {
  long long g = (total + bd - 1) / bd;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

inline long long chunk_rows(long long n, int nblk) { return (n + nblk - 1) / nblk; }

#define LGP_LAUNCH_CHECK(ctx)                 \
  do {                                        \
    ++(ctx)->launches;                        \
    LGP_CUDA_CHECK(cudaGetLastError());       \
  } while (0)

}  // namespace

int reduce_blocks(int64_t n, int t) {
  (void)t;
  long long b = (n + kRowsPerBlock - 1) / kRowsPerBlock;
  if (b > kMaxBlocks) b = kMaxBlocks;
  if (b < 1) b = 1;
  return (int)b;
}

void pack_rhs(Context* c, const double* V, int64_t n, int t, int64_t n_pad, int tb, int n_pass,
              double* out, const int* done) {
  k_pack<<<grid_for((long long)n_pass * n_pad * tb), 256, 0, c->stream>>>(V, n, t, n_pad, tb,
                                                                         n_pass, out, done);
  LGP_LAUNCH_CHECK(c);
}

void pack_rhs_tc(Context* c, const double* V, int64_t n, int t, int n_tiles, int tbn, int n_pass,
                 void* out, float* scale, int* inexact, const int* done) {
  // colmax scratch: the first t slots of `scale` reinterpreted would alias, so
  // the maxima live behind the inexact flag's 16-byte slot (see MatvecOp)
  unsigned long long* colmax = reinterpret_cast<unsigned long long*>(inexact + 4);
  LGP_CUDA_CHECK(cudaMemsetAsync(colmax, 0, (size_t)n_pass * tbn * 8, c->stream));
  if (t <= 256)
    k_colmax<<<grid_for(n * t / 4 + 1), reduce_bd(t), 0, c->stream>>>(V, n, t, colmax, done);
  else
    k_colmax_wide<<<dim3((t + 255) / 256, 64), 256, 0, c->stream>>>(V, n, t, colmax, done);
  LGP_LAUNCH_CHECK(c);
  k_colscale<<<1, 256, 0, c->stream>>>(colmax, t, n_pass * tbn, scale, done);
  LGP_LAUNCH_CHECK(c);
  LGP_CUDA_CHECK(cudaMemsetAsync(inexact, 0, sizeof(int), c->stream));
  k_pack_tc<<<grid_for((long long)n_pass * n_tiles * tbn * 64), 256, 0, c->stream>>>(
      V, n, t, n_tiles, tbn, n_pass, scale, (__half*)out, inexact, done);
  LGP_LAUNCH_CHECK(c);
}

void tcsym_epilogue(Context* c, const double* rowpart, const double* colpart, const int* r_ptr,
                    const int* r_rec, const int* c_ptr, const int* c_rec, int64_t n, double scale,
                    double noise, const double* noise_v, double* out, const int* done) {
  if (n <= 0) return;
  k_tcsym_epilogue<<<(unsigned)((n + 63) / 64), 64 * kTsGroups, 0, c->stream>>>(
      rowpart, colpart, r_ptr, r_rec, c_ptr, c_rec, n, scale, noise, noise_v, out, done);
  LGP_LAUNCH_CHECK(c);
}

void epilogue(Context* c, const double* partial, int n_seg, int n_pass, int64_t rows_pad, int tb,
              int64_t n_rows, int t, double scale, double noise, const double* noise_v,
              double* out, const int* done) {
  k_epilogue<<<grid_for(n_rows * t), 256, 0, c->stream>>>(
      partial, n_seg, n_pass, rows_pad, tb, n_rows, t, scale, noise, noise_v, out, done);
  LGP_LAUNCH_CHECK(c);
}

void sym_epilogue(Context* c, const double* rowp, const double* colp, int nb, int rb, int n_pass,
                  int tb, int64_t n, int t, double scale, double noise, const double* noise_v,
                  double* out, const int* done) {
  k_sym_epilogue<<<grid_for(n * t), 256, 0, c->stream>>>(rowp, colp, nb, rb, n_pass, tb, n, t,
                                                         scale, noise, noise_v, out, done);
  LGP_LAUNCH_CHECK(c);
}

void point_stats(Context* c, const double* x, int64_t n, int d, double* ctr, double* scratch,
                 double* stats) {
  // stats (device, d + 2 doubles): [mean (d) | max squared radius | non-finite flag]
  const int nblk = reduce_blocks(n, 1);
  const long long rows = chunk_rows(n, nblk);
  int* bad = reinterpret_cast<int*>(stats + d + 1);
  LGP_CUDA_CHECK(cudaMemsetAsync(stats, 0, (size_t)(d + 2) * sizeof(double), c->stream));
  if (n > 0) {
    k_pt_colsum<<<dim3(nblk, d), 256, 0, c->stream>>>(x, n, d, rows, scratch, bad);
    LGP_LAUNCH_CHECK(c);
  }
  k_pt_center<<<1, 512, 0, c->stream>>>(scratch, n > 0 ? nblk : 0, d, n, ctr, stats);
  LGP_LAUNCH_CHECK(c);
  if (n > 0) {
    k_pt_radius<<<grid_for(n), 256, 0, c->stream>>>(
        x, n, d, ctr, reinterpret_cast<unsigned long long*>(stats + d));
    LGP_LAUNCH_CHECK(c);
  }
}

void dot_partial(Context* c, const double* a, const double* b, int64_t n, int t, double* part,
                 const int* done) {
  const int nb = reduce_blocks(n, t);
  k_dot_partial<<<nb, reduce_bd(t), 0, c->stream>>>(a, b, n, t, chunk_rows(n, nb), part, done);
  LGP_LAUNCH_CHECK(c);
}

void dot_final(Context* c, const double* part, int nblk, int t, double* out, const int* done) {
  k_dot_final<<<1, 256, 0, c->stream>>>(part, nblk, t, out, done);
  LGP_LAUNCH_CHECK(c);
}

void add_inplace(double* dst, const double* src, int64_t n, cudaStream_t stream) {
  if (n <= 0) return;
  k_add_inplace<<<grid_for(n), 256, 0, stream>>>(dst, src, n);
  LGP_CUDA_CHECK(cudaGetLastError());
}

void fill(Context* c, double* p, int64_t n, double v) {
  k_fill<<<grid_for(n), 256, 0, c->stream>>>(p, n, v);
  LGP_LAUNCH_CHECK(c);
}

void cg_init(Context* c, const double* b, double* x, double* r, double* p, int64_t n, int t,
             double rel_tol, const double* bb_final, CgState s) {
  k_cg_init_vecs<<<grid_for(n * t), 256, 0, c->stream>>>(b, x, r, p, n * t);
  LGP_LAUNCH_CHECK(c);
  k_cg_init_scalars<<<1, 256, 0, c->stream>>>(bb_final, t, rel_tol, s);
  LGP_LAUNCH_CHECK(c);
}

void cg_fin_pap(Context* c, const double* part, int nblk, int t, CgState s) {
  k_cg_fin_pap<<<1, 256, 0, c->stream>>>(part, nblk, t, s);
  LGP_LAUNCH_CHECK(c);
}

void cg_update_xr(Context* c, double* x, double* r, const double* p, const double* ap, int64_t n,
                  int t, CgState s, double* part) {
  const int nb = reduce_blocks(n, t);
  k_cg_update_xr<<<nb, reduce_bd(t), 0, c->stream>>>(x, r, p, ap, n, t, chunk_rows(n, nb), s, part);
  LGP_LAUNCH_CHECK(c);
}

void cg_fin_rs(Context* c, const double* part, int nblk, int t, int it, int max_iter, CgState s) {
  k_cg_fin_rs<<<1, 256, 0, c->stream>>>(part, nblk, t, it, max_iter, s);
  LGP_LAUNCH_CHECK(c);
}

void cg_update_p(Context* c, double* p, const double* r, int64_t n, int t, CgState s) {
  k_cg_update_p<<<grid_for(n * t), 256, 0, c->stream>>>(p, r, n * t, t, s);
  LGP_LAUNCH_CHECK(c);
}

void cg1_pack(Context* c, double* p, const double* r, double* vpack, int64_t n, int64_t n_pad,
              CgState s) {
  k_cg1_pack<<<grid_for(n_pad), 256, 0, c->stream>>>(p, r, vpack, n, n_pad, s);
  LGP_LAUNCH_CHECK(c);
}

void tcsym_epilogue_cg(Context* c, const double* rowpart, const double* colpart, const int* r_ptr,
                       const int* r_rec, const int* c_ptr, const int* c_rec, int64_t n,
                       double scale, double noise, const double* p, double* out, double* part,
                       unsigned* counter, CgState s) {
  if (n <= 0) return;
  k_tcsym_epilogue_cg<<<(unsigned)((n + 63) / 64), 64 * kTsGroups, 0, c->stream>>>(
      rowpart, colpart, r_ptr, r_rec, c_ptr, c_rec, n, scale, noise, p, out, part, counter, s);
  LGP_LAUNCH_CHECK(c);
}

void cg1_vec(Context* c, const double* rowpart, const double* colpart, const int* r_ptr,
             const int* r_rec, const int* c_ptr, const int* c_rec, int64_t n, int64_t n_pad, double scale,
             double noise, double* x, double* r, double* p, double* ap, double* vpack, double* part_pap,
             double* part_rs, unsigned* bar, int it, int max_iter, CgState s,
             unsigned long long* trace) {
  if (n <= 0) return;
  int nvb = cg1_blocks(n);
  long long n_ll = n, npad_ll = n_pad;
  void* args[] = {(void*)&rowpart, (void*)&colpart, (void*)&r_ptr, (void*)&r_rec, (void*)&c_ptr,
                  (void*)&c_rec, (void*)&n_ll, (void*)&npad_ll, (void*)&scale, (void*)&noise,
                  (void*)&x, (void*)&r, (void*)&p, (void*)&ap, (void*)&vpack, (void*)&part_pap,
                  (void*)&part_rs, (void*)&nvb, (void*)&bar, (void*)&it, (void*)&max_iter, (void*)&s,
                  (void*)&trace};
  // one CTA per SM, and enough virtual 256-thread blocks per CTA
  const int grid = std::max(c->sm_count, (nvb + kVecThreads / 256 - 1) / (kVecThreads / 256));
  LGP_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_cg1_vec, dim3((unsigned)grid),
                                             dim3(kVecThreads), args, 0, c->stream));
}

int cg1_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 4, (n + 255) / 256)); }

bool cg1_vec_supported(Context* c, int64_t n) {
  // the grid barrier needs every CTA resident at once (cooperative launch)
  int coop = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->device) != cudaSuccess || !coop) {
    cudaGetLastError();
    return false;
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg1_vec, kVecThreads, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const int nvb = cg1_blocks(n);
  const int grid = std::max(c->sm_count, (nvb + kVecThreads / 256 - 1) / (kVecThreads / 256));
  return (int64_t)per_sm * c->sm_count >= grid;
}

void cg1_pap(Context* c, const double* p, const double* ap, int64_t n, double* part,
             unsigned* counter, CgState s) {
  k_cg1_pap<<<(unsigned)((n + 63) / 64), 64, 0, c->stream>>>(p, ap, n, part, counter, s);
  LGP_LAUNCH_CHECK(c);
}

void cg1_update(Context* c, double* x, double* r, const double* p, const double* ap, int64_t n,
                double* part, unsigned* counter, int it, int max_iter, CgState s) {
  k_cg1_update<<<cg1_blocks(n), 256, 0, c->stream>>>(x, r, p, ap, n, part, counter, it, max_iter, s);
  LGP_LAUNCH_CHECK(c);
}

void cg_shift_init(Context* c, const double* b, int64_t n, int nsh, double* xs, double* ps,
                   CgShiftState* st) {
  k_cg_shift_init<<<grid_for(n * nsh), 256, 0, c->stream>>>(b, n, nsh, xs, ps, st);
  LGP_LAUNCH_CHECK(c);
}

void cg_shift(Context* c, double* xs, double* ps, const double* r, int64_t n, int nsh,
              const double* sig, CgShiftState* st, CgState s, int it) {
  k_cg_shift<<<grid_for(n * nsh), 256, 0, c->stream>>>(xs, ps, r, n, nsh, sig, st, s, it);
  LGP_LAUNCH_CHECK(c);
}

void gather_cols(Context* c, const double* src, int64_t n, int t, const int* map, int t_run,
                 double* dst, const int* done) {
  k_gather_cols<<<grid_for(n * t_run), 256, 0, c->stream>>>(src, n, t, map, t_run, dst, done);
  LGP_LAUNCH_CHECK(c);
}

void scatter_cols(Context* c, const double* src, int64_t n, int t_run, const int* map, int t,
                  double* dst, const int* done) {
  k_scatter_cols<<<grid_for(n * t_run), 256, 0, c->stream>>>(src, n, t_run, map, t, dst, done);
  LGP_LAUNCH_CHECK(c);
}

void lz_init(Context* c, const double* z, double* q0, int64_t n, int t, const double* zz_final,
             LzState s) {
  k_lz_init<<<grid_for(n * t), 256, 0, c->stream>>>(z, q0, n * t, t, zz_final);
  LGP_LAUNCH_CHECK(c);
  k_lz_init_scalars<<<1, 256, 0, c->stream>>>(zz_final, t, s);
  LGP_LAUNCH_CHECK(c);
}

void lz_fin_alpha(Context* c, const double* part, int nblk, int t, int j, int steps, LzState s) {
  k_lz_fin_alpha<<<1, 256, 0, c->stream>>>(part, nblk, t, j, steps, s);
  LGP_LAUNCH_CHECK(c);
}

void lz_update1(Context* c, double* w, const double* q, const double* qprev, int64_t n, int t,
                int j, int steps, LzState s) {
  k_lz_update1<<<grid_for(n * t), 256, 0, c->stream>>>(w, q, qprev, n * t, t, j, steps, s);
  LGP_LAUNCH_CHECK(c);
}

void lz_multidot(Context* c, const double* basis, int64_t stride, int nb, const double* w,
                 int64_t n, int t, double* part, const int* done) {
  const int nblk = reduce_blocks(n, t);
  if (2 * t <= 256) {
    const int kb = 256 / t;
    k_lz_multidot2<<<dim3(nblk, (nb + kb - 1) / kb), kb * t, 0, c->stream>>>(
        basis, stride, nb, w, n, t, chunk_rows(n, nblk), part, done);
  } else {
    k_lz_multidot<<<nblk, reduce_bd(t), 0, c->stream>>>(basis, stride, nb, w, n, t,
                                                        chunk_rows(n, nblk), part, done);
  }
  LGP_LAUNCH_CHECK(c);
}

void lz_fin_h(Context* c, const double* part, int nblk, int nb, int t, LzState s) {
  k_lz_fin_h<<<(nb * t + 31) / 32, 256, 0, c->stream>>>(part, nblk, nb, t, s);
  LGP_LAUNCH_CHECK(c);
}

void lz_update2(Context* c, double* w, const double* basis, int64_t stride, int nb, int64_t n,
                int t, LzState s, double* part) {
  const int nblk = reduce_blocks(n, t);
  k_lz_update2<<<nblk, reduce_bd(t), 0, c->stream>>>(w, basis, stride, nb, n, t,
                                                     chunk_rows(n, nblk), s, part);
  LGP_LAUNCH_CHECK(c);
}

void lz_fin_beta(Context* c, const double* part, int nblk, int t, int j, int steps, LzState s) {
  k_lz_fin_beta<<<1, 256, 0, c->stream>>>(part, nblk, t, j, steps, s);
  LGP_LAUNCH_CHECK(c);
}

void lz_normalize(Context* c, const double* w, double* qnext, int64_t n, int t, LzState s) {
  k_lz_normalize<<<grid_for(n * t), 256, 0, c->stream>>>(w, qnext, n * t, t, s);
  LGP_LAUNCH_CHECK(c);
}

void quad_dot(Context* c, const double* a, const double* b, int64_t n, int t, double* part,
              double* out) {
  dot_partial(c, a, b, n, t, part, nullptr);
  dot_final(c, part, reduce_blocks(n, t), t, out, nullptr);
}

}  // namespace vec
}  // namespace lgp

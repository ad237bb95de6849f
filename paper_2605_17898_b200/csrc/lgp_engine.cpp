// Matvec engine (feature prep -> fused K1 -> FP64 epilogue) and the
// device-resident CG / Lanczos drivers.
//
// Multi-GPU (world > 1): rank g owns rows [g*S, min((g+1)*S, n)) of K with
// S = ceil(n/world); X is replicated. Each iteration computes the local rows
// of the product, all-gathers the slices in place (one NCCL call over
// NVLink), and then runs the FP64 vector updates redundantly on the full
// vectors. All ranks hold bit-identical state, the host loop's stop decision
// is identical on every rank, and no scalar all-reduce is needed.
#include <algorithm>
#include <functional>
#include <vector>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "lgp_internal.h"

namespace lgp {

void Context::activate() { LGP_CUDA_CHECK(cudaSetDevice(device)); }

size_t Context::pool_round(size_t bytes) {
  size_t r = 4096;
  while (r < bytes) r <<= 1;
  return r;
}

void* Context::pool_get(size_t bytes) {
  const size_t r = pool_round(bytes);
  auto& v = pool[r];
  if (!v.empty()) {
    void* p = v.back();
    v.pop_back();
    return p;
  }
  void* p = nullptr;
  LGP_CUDA_CHECK(cudaMalloc(&p, r));
  return p;
}

void Context::pool_put(void* p, size_t bytes) {
  if (p) pool[pool_round(bytes)].push_back(p);
}

void* Context::scratch_get(const std::string& name, size_t bytes) {
  if (bytes == 0) bytes = 16;
  DeviceBuffer& b = scratch[name];
  if (b.bytes < bytes) {
    if (b.ptr) {
      LGP_CUDA_CHECK(cudaStreamSynchronize(stream));
      LGP_CUDA_CHECK(cudaFree(b.ptr));
      b.ptr = nullptr;
      b.bytes = 0;
    }
    const size_t want = bytes + bytes / 8;  // growth slack
    LGP_CUDA_CHECK(cudaMalloc(&b.ptr, want));
    b.bytes = want;
  }
  return b.ptr;
}

namespace {
// scratch budget of the symmetric kernels' partials; larger operators use the
// plain row-block kernels (partials O(N) per column segment)
constexpr double kSymPartialBudget = 16.0 * (1ull << 30);

int pick_tb(int t) {
  if (t >= 16) return 16;
  int tb = 1;
  while (tb < t) tb <<= 1;
  return tb;
}
template <class T>
T ceil_div(T a, T b) {
  return (a + b - 1) / b;
}
// pairs (I, c) with c >= 2I of a rectangle of the (row block, chunk) grid
int64_t ts_pairs(int Ia, int Ib, int ca, int cb) {
  int64_t p = 0;
  for (int I = Ia; I < Ib; ++I) p += std::max(0, cb - std::max(ca, 2 * I));
  return p;
}
// list-scheduling model: items dispatched in order onto the free-earliest SM;
// cost ~ pairs + a row-switch and an item overhead (in pair units)
double ts_makespan(const std::vector<TsRect>& v, int slots) {
  std::vector<double> sm(std::max(1, slots), 0.0);
  std::make_heap(sm.begin(), sm.end(), std::greater<double>());
  for (const TsRect& r : v) {
    std::pop_heap(sm.begin(), sm.end(), std::greater<double>());
    sm.back() += (double)r.pairs + 1.0 * (r.Ib - r.Ia) + 4.0;
    std::push_heap(sm.begin(), sm.end(), std::greater<double>());
  }
  return *std::max_element(sm.begin(), sm.end());
}
}  // namespace

std::vector<TsRect> ts_items(int n_rb, int n_tiles, int R, int slots) {
  std::vector<TsRect> base;
  const int nG = (int)ceil_div<int64_t>(n_rb, R);
  auto add = [&](std::vector<TsRect>& v, int Ia, int Ib, int ca, int cb) {
    Ib = std::min(Ib, n_rb);
    cb = std::min(cb, n_tiles);
    if (Ia >= Ib || ca >= cb) return;
    const int64_t p = ts_pairs(Ia, Ib, ca, cb);
    if (p > 0) v.push_back(TsRect{Ia, Ib, ca, cb, p});
  };
  for (int d = 1; d < nG; ++d)
    for (int gi = 0; gi + d < nG; ++gi) add(base, gi * R, (gi + 1) * R, 2 * (gi + d) * R, 2 * (gi + d + 1) * R);
  for (int gi = 0; gi < nG; ++gi) add(base, gi * R, (gi + 1) * R, 2 * gi * R, 2 * (gi + 1) * R);
  // quarters for the items that start within the last two waves of work
  int64_t total = 0, big = 1;
  for (const TsRect& r : base) {
    total += r.pairs;
    big = std::max(big, r.pairs);
  }
  const int64_t tail = 2 * (int64_t)std::max(1, slots) * big;
  std::vector<TsRect> out;
  int64_t acc = 0;
  for (const TsRect& r : base) {
    if (R > 1 && total - acc <= tail) {
      const int Im = (r.Ia + r.Ib + 1) / 2, cm = (r.ca + r.cb + 1) / 2;
      add(out, r.Ia, Im, r.ca, cm);
      add(out, r.Ia, Im, cm, r.cb);
      add(out, Im, r.Ib, r.ca, cm);
      add(out, Im, r.Ib, cm, r.cb);
    } else {
      out.push_back(r);
    }
    acc += r.pairs;
  }
  std::stable_sort(out.begin(), out.end(), [](const TsRect& x, const TsRect& y) { return x.pairs > y.pairs; });
  return out;
}

namespace {
void launch(Context* ctx, CUfunction f, unsigned gx, unsigned gy, unsigned bx, size_t smem,
            void* args) {
  void* params[] = {args};
  LGP_CU_CHECK(drv::LaunchKernel(f, gx, gy, 1, bx, 1, 1, (unsigned)smem, (CUstream)ctx->stream,
                              params, nullptr));
  ++ctx->launches;
}
}  // namespace

// K1-TC-sym work schedule for an n_rb x n_tiles square operator (host
// side; cached per context: the list-scheduling model and the record lists
// cost milliseconds at N ~ 1e5 and the CG / Lanczos drivers prepare per call)
const TsSchedule& ts_schedule(Context* ctx, int n_rb, int n_tiles, int rmax, bool rank_split) {
  const char* fe = std::getenv("LGP_TS_R");
  const std::string key = std::to_string(n_rb) + "/" + std::to_string(n_tiles) + "/" + std::to_string(rmax) +
                      "/" + std::to_string(rank_split && ctx->world > 1 ? ctx->world : 1) + "/" +
                      std::to_string(ctx->rank) + "/" + (fe ? fe : "");
  auto hit = ctx->ts_cache.find(key);
  if (hit != ctx->ts_cache.end()) return *hit->second;
  auto out = std::make_shared<TsSchedule>();
  TsSchedule& S = *out;
  // work items: rectangles of the (row block, chunk) triangle c >= 2I -
  // R x 2R super-tiles (full ones first, the diagonal ones after), the
  // ones dispatched in the last two waves split into quarters; R picked
  // by a list-scheduling model of the items on the SMs (one CTA per SM)
  // so the items fill whole waves while the scratch (R x 128 + 2R x 64
  // doubles per item) stays O(N)
  int R = 1;
  std::vector<TsRect> rects;
  {
    const int cands[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64};
    double best = 1e300;
    int forced = 0;
    if (const char* e = std::getenv("LGP_TS_R")) forced = std::max(1, std::min(rmax, atoi(e)));
    for (int Rc : cands) {
      if (forced) Rc = forced;  // LGP_TS_R: exactly that R (any value <= rmax)
      else if (Rc > rmax) break;
      const int64_t nG = ceil_div<int64_t>(n_rb, Rc);
      if (nG * (nG + 1) / 2 > 2000000) continue;
      std::vector<TsRect> rc = ts_items(n_rb, n_tiles, Rc, ctx->sm_count);
      const double span = ts_makespan(rc, ctx->sm_count);
      if (span < best * 0.995) {  // near-ties: the larger R (less scratch)
        best = span;
        R = Rc;
        rects.swap(rc);
      } else if (span <= best * 1.005) {
        R = Rc;
        rects.swap(rc);
      }
      if (forced) break;
    }
    if (forced) R = forced;
  }
  if (rects.empty()) throw Error(LGP_E_UNSUPPORTED, "K1-TC-sym: no work items");
  const int n_items = (int)rects.size();
  int item_lo = 0, item_hi = n_items;
  if (rank_split && ctx->world > 1) {
    // contiguous item ranges with (nearly) equal pair counts per rank
    int64_t total = 0;
    for (const TsRect& r : rects) total += r.pairs;
    int64_t acc = 0;
    int r = 0;
    std::vector<int> cut(ctx->world + 1, n_items);
    cut[0] = 0;
    for (int q = 0; q < n_items; ++q) {
      while (r < ctx->world - 1 && acc >= (int64_t)(r + 1) * total / ctx->world) cut[++r] = q;
      acc += rects[q].pairs;
    }
    item_lo = cut[ctx->rank];
    item_hi = cut[ctx->rank + 1];
  }
  // item table (Ia, Ib, ca, cb, first row record, first chunk record) +
  // the records each row block / chunk sums (this rank's items, in item
  // order: the epilogue's fixed summation order)
  std::vector<int> it((size_t)n_items * 6);
  std::vector<std::vector<int>> rl(n_rb), cl(n_tiles);
  int nrr = 0, ncr = 0;
  for (int q = 0; q < n_items; ++q) {
    const TsRect& r = rects[q];
    it[6 * q] = r.Ia;
    it[6 * q + 1] = r.Ib;
    it[6 * q + 2] = r.ca;
    it[6 * q + 3] = r.cb;
    it[6 * q + 4] = nrr;
    it[6 * q + 5] = ncr;
    if (q < item_lo || q >= item_hi) continue;
    for (int I = r.Ia; I < r.Ib; ++I) rl[I].push_back(nrr++);
    for (int c = r.ca; c < r.cb; ++c) cl[c].push_back(ncr++);
  }
  std::vector<int> idx;
  idx.reserve((size_t)n_rb + n_tiles + 2 + nrr + ncr);
  idx.push_back(0);
  for (int I = 0; I < n_rb; ++I) idx.push_back(idx.back() + (int)rl[I].size());
  idx.push_back(0);
  for (int c = 0; c < n_tiles; ++c) idx.push_back(idx.back() + (int)cl[c].size());
  for (int I = 0; I < n_rb; ++I) idx.insert(idx.end(), rl[I].begin(), rl[I].end());
  for (int c = 0; c < n_tiles; ++c) idx.insert(idx.end(), cl[c].begin(), cl[c].end());
  S.R = R;
  S.n_items = n_items;
  S.item_lo = item_lo;
  S.item_hi = item_hi;
  S.nrr = nrr;
  S.ncr = ncr;
  S.it.swap(it);
  S.idx.swap(idx);
  ctx->ts_cache[key] = out;
  return S;
}

void MatvecOp::prepare() {
  int tb = pick_tb(t);
  {
    // wide point sets: the norm trick's cancellation would cost accuracy
    double c2 = 0.0;
    for (int j = 0; j < rows->d; ++j) {
      const double e = rows->center[j] - cols->center[j];
      c2 += e * e;
    }
    const double reach = rows->radius + cols->radius + std::sqrt(c2);
    if (r2_gain(k->tree) * reach * reach > kNormTrickReach2) {
      allow_tc = false;
      flags |= LGP_DIST_DIRECT;
    }
  }
  // the CG matvec (square operator, one RHS): symmetric tensor-core kernel,
  // each unordered pair evaluated once, FP64 contraction with the exact p -
  // exactly symmetric, so CG iteration counts match the SIMT kernel. Its
  // scratch is O(N) (super-tiles, see prepare below), so the choice depends on
  // the tree and flags only: identical on every rank of a multi-rank CG.
  tcsym = false;
  if (t == 1 && rows == cols && (!ctx->sharded() || rank_split) && row0 == 0 && n_rows == rows->n &&
      !(flags & (LGP_NO_SYM | LGP_FORCE_SIMT | LGP_DIST_DIRECT)) && !std::getenv("LGP_NO_TCSYM")) {
    Plan p = make_tc_plan(k->tree, rows->d, 16, flags);
    if (p.tc && p.ts_rmax >= 1) {
      plan = p;
      tcsym = true;
    }
  }
  if (!tcsym && allow_tc) {
    plan = make_tc_plan(k->tree, rows->d, std::max(t, tc_t_hint), flags);
    // many Periodic features (> 24 per point) spill in the multi-RHS
    // epilogue: the SIMT kernel is faster there (2 leaves at D = 8: 2.97 vs
    // 3.59 ms; tools/periodic_pf_sweep.py); the t = 1 symmetric kernel still wins
    if (plan.tc && plan.tc_pf > 24) plan.tc = false;
  }
  if (plan.tc) {
    tb = plan.tc_n;
  } else {
    plan = make_plan(k->tree, rows->d, tb, flags);
  }
  mod = get_module(ctx, plan);
  const Tuning& tu = plan.tune;
  const int rows_per_cta = plan.tc ? 128 : tu.threads * tu.r;
  n_rb = (int)ceil_div<int64_t>(std::max<int64_t>(n_rows, 1), rows_per_cta);
  n_rows_pad = n_rb * rows_per_cta;
  const int cc = plan.tc ? 64 : tu.cc;
  n_tiles = (int)ceil_div<int64_t>(std::max<int64_t>(cols->n, 1), cc);
  n_cols_pad = n_tiles * cc;
  n_pass = ceil_div(t, tb);

  // Column split so that (row blocks x segments x passes) CTAs fill whole
  // waves of resident CTAs: minimise waves / segments (+ partial traffic).
  const int slots = ctx->sm_count * mod->blocks_per_sm;
  const int64_t base = (int64_t)n_rb * n_pass;
  int best = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= std::min(n_tiles, 64); ++s) {
    const int64_t items = base * s;
    const double waves = (double)ceil_div<int64_t>(items, slots);
    const double cost = waves / s + 0.002 * s;
    if (cost < best_cost - 1e-12) {
      best_cost = cost;
      best = s;
    }
  }
  if (const char* e = std::getenv("LGP_SEGMENTS")) best = std::max(1, std::min(n_tiles, atoi(e)));
  tiles_per_seg = ceil_div(n_tiles, best);
  if (tiles_per_seg_hint > 0) tiles_per_seg = std::min(n_tiles, tiles_per_seg_hint);
  n_seg = ceil_div(n_tiles, tiles_per_seg);

  if (!tcsym) partial = (double*)ctx->scratch_get(tag + ".part", (size_t)n_seg * n_pass * n_rows_pad * tb * 8);
  if (plan.tc) {
    // operands pre-tiled in the UMMA canonical layout, FP16 hi/lo split
    fr = (float*)ctx->scratch_get(tag + ".a1", (size_t)n_rows_pad * plan.tc_kd * 2);
    fc = (float*)ctx->scratch_get(tag + ".b1", (size_t)n_cols_pad * plan.tc_kd * 2);
    if (plan.tc_pf > 0) {
      r32 = (float*)ctx->scratch_get(tag + ".r32", (size_t)n_rows_pad * plan.tc_fw * 4);
      c32 = (float*)ctx->scratch_get(tag + ".c32", (size_t)n_cols_pad * plan.tc_fw * 4);
    }
    vtc = ctx->scratch_get(tag + ".vtc", (size_t)n_pass * n_cols_pad * 2 * tb * 2);
    vscale = (float*)ctx->scratch_get(tag + ".vscale", (size_t)2 * n_pass * tb * 4);  // [part][pass][tb]
    // inexact flag (16 B) followed by the per-column max |V| used for the scales
    v_inexact = (int*)ctx->scratch_get(tag + ".vflag", 16 + (size_t)n_pass * tb * 8);
    LgpPrepArgs pa = plan.prep;
    pa.x = rows->x;
    pa.ctr = cols->ctr;
    pa.fr = fr;
    pa.fc = fc;
    pa.f32 = r32;
    pa.row0 = row0;
    pa.n = n_rows;
    pa.n_pad = n_rows_pad;
    int tile_rows = 128, is_col = 0;
    void* p1[] = {&pa, &tile_rows, &is_col};
    LGP_CU_CHECK(drv::LaunchKernel(mod->prep, (unsigned)ceil_div<int64_t>(n_rows_pad, 128), 1, 1,
                                   128, 1, 1, 0, (CUstream)ctx->stream, p1, nullptr));
    ++ctx->launches;
    LgpPrepArgs pc = plan.prep;
    pc.x = cols->x;
    pc.ctr = cols->ctr;
    pc.fr = fr;
    pc.fc = fc;
    pc.f32 = c32;
    pc.row0 = 0;
    pc.n = cols->n;
    pc.n_pad = n_cols_pad;
    int tile_cols = 64, is_col1 = 1;
    void* p2[] = {&pc, &tile_cols, &is_col1};
    LGP_CU_CHECK(drv::LaunchKernel(mod->prep, (unsigned)ceil_div<int64_t>(n_cols_pad, 128), 1, 1,
                                   128, 1, 1, 0, (CUstream)ctx->stream, p2, nullptr));
    ++ctx->launches;
    if (tcsym) {
      const TsSchedule& sc = ts_schedule(ctx, n_rb, n_tiles, plan.ts_rmax, rank_split);
      n_items = sc.n_items;
      ts_R = sc.R;
      item_lo = sc.item_lo;
      item_hi = sc.item_hi;
      const int nrr = sc.nrr, ncr = sc.ncr;
      const std::vector<int>& it = sc.it;
      const std::vector<int>& idx = sc.idx;
      items = (int*)ctx->scratch_get(tag + ".items", it.size() * 4);
      recs = (int*)ctx->scratch_get(tag + ".recs", idx.size() * 4);
      // [n_rb + 1] row pointers | [n_tiles + 1] chunk pointers | row records | chunk records
      r_ptr = recs;
      c_ptr = recs + n_rb + 1;
      r_rec = c_ptr + n_tiles + 1;
      c_rec = r_rec + nrr;
      // pageable sources: the copies complete before cudaMemcpyAsync returns
      LGP_CUDA_CHECK(cudaMemcpyAsync(items, it.data(), it.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
      LGP_CUDA_CHECK(cudaMemcpyAsync(recs, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
      // partials of this rank's items only: one 128-row record per (item, row
      // block), one 64-column record per (item, chunk)
      partial = (double*)ctx->scratch_get(tag + ".rowp", (size_t)std::max(nrr, 1) * 128 * 8);
      colpart = (double*)ctx->scratch_get(tag + ".colp", (size_t)std::max(ncr, 1) * 64 * 8);
      vpack = (double*)ctx->scratch_get(tag + ".v", (size_t)std::max(n_rows_pad, n_cols_pad) * 8);
    }
    return;
  }
  // symmetric block-pair kernel for the square operator on a single rank
  // block-pair partials: 2 x rows_per_cta FP64 per unit, n_rb^2 / 2 units
  const double sym_bytes = (double)n_rb * (n_rb + 1) / 2.0 * rows_per_cta * 16.0 * n_pass * tb;
  // (and enough block pairs to fill the GPU: small operators take the plain
  // kernel, whose column segments supply the parallelism)
  sym = (rows == cols) && !ctx->sharded() && tb == 1 && !(flags & LGP_NO_SYM) &&
        (rows_per_cta % tu.cc) == 0 && (int64_t)n_rb * (n_rb + 1) / 2 >= 2 * ctx->sm_count &&
        sym_bytes <= kSymPartialBudget;
  if (sym) {
    n_cols_pad = n_rows_pad;  // column blocks = row blocks
    n_tiles = n_cols_pad / tu.cc;
    n_units = n_rb * (n_rb + 1) / 2;
    std::vector<int> tab((size_t)n_units * 2);
    int u = 0;
    for (int I = 0; I < n_rb; ++I)
      for (int J = I; J < n_rb; ++J) {
        tab[2 * u] = I;
        tab[2 * u + 1] = J;
        ++u;
      }
    units = (int*)ctx->scratch_get(tag + ".units", tab.size() * 4);
    LGP_CUDA_CHECK(cudaMemcpyAsync(units, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice,
                                   ctx->stream));
    const size_t pb = (size_t)n_units * n_pass * rows_per_cta * tb * 8;
    partial = (double*)ctx->scratch_get(tag + ".part", pb);
    colpart = (double*)ctx->scratch_get(tag + ".colp", pb);
    smem_sym = plan.smem_bytes + (size_t)(tu.threads / 32) * tu.cc * tb * 8;
  }
  fr = (float*)ctx->scratch_get(tag + ".fr", (size_t)n_rows_pad * plan.fr * 4);
  fc = (float*)ctx->scratch_get(tag + ".fc", (size_t)n_cols_pad * plan.fc * 4);
  vpack = (double*)ctx->scratch_get(tag + ".v", (size_t)n_pass * n_cols_pad * tb * 8);

  // features of the local rows and of all columns, centred on the column set
  LgpPrepArgs pa = plan.prep;
  pa.x = rows->x;
  pa.ctr = cols->ctr;
  pa.fr = fr;
  pa.fc = nullptr;
  pa.row0 = row0;
  pa.n = n_rows;
  pa.n_pad = n_rows_pad;
  launch(ctx, mod->prep, (unsigned)ceil_div<int64_t>(n_rows_pad, 128), 1, 128, 0, &pa);
  LgpPrepArgs pc = plan.prep;
  pc.x = cols->x;
  pc.ctr = cols->ctr;
  pc.fr = nullptr;
  pc.fc = fc;
  pc.row0 = 0;
  pc.n = cols->n;
  pc.n_pad = n_cols_pad;
  launch(ctx, mod->prep, (unsigned)ceil_div<int64_t>(n_cols_pad, 128), 1, 128, 0, &pc);
}

// per-launch CUDA events around the fused K1 kernel (lgp_ctx_set_profile)
std::pair<cudaEvent_t, cudaEvent_t> k1_event_begin(Context* ctx) {
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (!ctx->profile) return ev;
  if (ctx->ev_pool.empty()) {
    LGP_CUDA_CHECK(cudaEventCreate(&ev.first));
    LGP_CUDA_CHECK(cudaEventCreate(&ev.second));
  } else {
    ev = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
  }
  LGP_CUDA_CHECK(cudaEventRecord(ev.first, ctx->stream));
  return ev;
}

void k1_event_end(Context* ctx, std::pair<cudaEvent_t, cudaEvent_t> ev) {
  if (!ctx->profile || !ev.first) return;
  LGP_CUDA_CHECK(cudaEventRecord(ev.second, ctx->stream));
  ctx->ev_pending.push_back(ev);
}

void MatvecOp::tcsym_kernel(const int* done) {
  LgpTcSymArgs a;
  std::memset(&a, 0, sizeof a);
  a.a1 = fr;
  a.b1 = fc;
  a.v = vpack;
  a.r32 = r32;
  a.c32 = c32;
  a.items = items;
  a.rowpart = partial;
  a.colpart = colpart;
  a.done = done;
  a.item_base = item_lo;
  a.R = ts_R;
  a.n_rb = n_rb;
  a.n_tiles = n_tiles;
  std::memcpy(a.kc, plan.tca.kc, sizeof a.kc);
  if (item_hi > item_lo)
    launch(ctx, mod->tcsym, (unsigned)(item_hi - item_lo), 1, 64 + 128 * plan.ts_nwg,
           plan.smem_tcsym_fixed + (size_t)4096 * ts_R, &a);
}

// first column segment of V's second part (own column scales): half the
// segments with one RHS pass and >= 2 segments, else n_seg (one part)
int MatvecOp::tc_split() const {
  if (n_pass != 1 || n_seg < 2) return n_seg;
  const int s = (n_seg + 1) / 2;
  // the second part must hold columns (trailing segments can be empty)
  return (int64_t)s * tiles_per_seg * 64 < cols->n ? s : n_seg;
}

bool MatvecOp::run_staged(const double* V_host, double* V_dev, double* out_dev, double noise,
                          bool square, const std::function<void()>& after_copy0) {
  if (!plan.tc || tcsym || n_pass != 1 || n_seg < 2) return false;
  const int tb = plan.tune.tb;
  if (!ctx->copy_stream) {
    LGP_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : ctx->copy_ev) LGP_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // V_dev is context scratch: earlier work on the main stream may still read it
  LGP_CUDA_CHECK(cudaEventRecord(ctx->copy_ev[1], ctx->stream));
  LGP_CUDA_CHECK(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_ev[1], 0));
  // two parts = the two runs of column segments that run() packs with their
  // own column scales (tc_split()), so both paths give the same bits
  const int s_split = tc_split();
  const int64_t ncols = cols->n;
  LgpTcArgs a = plan.tca;
  a.v_inexact = v_inexact;
  a.vscale = vscale;
  a.a1 = fr;
  a.b1 = fc;
  a.r32 = r32;
  a.c32 = c32;
  a.v = vtc;
  a.partial = partial;
  a.done = nullptr;
  a.n_rows_pad = n_rows_pad;
  a.n_rb = n_rb;
  a.n_pass = n_pass;
  a.tiles_per_seg = tiles_per_seg;
  a.n_tiles = n_tiles;
  for (int h = 0; h < 2; ++h) {
    const int s0 = h ? s_split : 0, s1 = h ? n_seg : s_split;
    const int64_t r0 = std::min<int64_t>((int64_t)s0 * tiles_per_seg * 64, ncols);
    const int64_t r1 = std::min<int64_t>((int64_t)s1 * tiles_per_seg * 64, ncols);
    if (s1 <= s0) continue;  // (tc_split: a second part always holds columns)
    LGP_CUDA_CHECK(cudaMemcpyAsync(V_dev + r0 * t, V_host + r0 * t, (size_t)(r1 - r0) * t * 8,
                                   cudaMemcpyHostToDevice, ctx->copy_stream));
    LGP_CUDA_CHECK(cudaEventRecord(ctx->copy_ev[h & 1], ctx->copy_stream));
    // the host-side V scan once every copy is queued, while the first part's
    // K1 runs (a pageable copy blocks the host, so scanning right after the
    // first copy would delay that K1); on failure nothing is returned and
    // the streams drain first (the caller may free V right away)
    if ((h == 1 || s_split >= n_seg) && after_copy0) {
      try {
        after_copy0();
      } catch (...) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamSynchronize(ctx->stream);
        throw;
      }
    }
    LGP_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, ctx->copy_ev[h & 1], 0));
    // per-part power-of-two column scales: the K1 undoes them per CTA, and a
    // power-of-two change only shifts the FP16 exponents
    const int tile0 = s0 * tiles_per_seg;
    vec::pack_rhs_tc(ctx, V_dev + r0 * t, r1 - r0, t, (int)ceil_div<int64_t>(r1 - r0, 64), tb, 1,
                     static_cast<char*>(vtc) + (size_t)tile0 * 2 * tb * 64 * 2, vscale + (h ? tb : 0),
                     v_inexact, nullptr);
    a.seg_base = s0;
    a.seg_split = s_split;
    a.n_seg = s1 - s0;
    const int64_t grid = (int64_t)n_rb * (s1 - s0) * n_pass;
    if (grid > 0x7fffffff) throw Error(LGP_E_UNSUPPORTED, "problem too large for one launch");
    auto ev = k1_event_begin(ctx);
    launch(ctx, mod->matvec, (unsigned)grid, 1, plan.tune.threads, plan.smem_bytes, &a);
    k1_event_end(ctx, ev);
  }
  vec::epilogue(ctx, partial, n_seg, n_pass, n_rows_pad, tb, n_rows, t, plan.root_scale, noise,
                square ? V_dev + row0 * t : nullptr, out_dev, nullptr);
  return true;
}

void MatvecOp::run(const double* V_dev, double* out_dev, double noise, const double* noise_v,
                   const int* done) {
  const int tb = plan.tune.tb;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  auto prof_begin = [&]() { ev = k1_event_begin(ctx); };
  auto prof_end = [&]() { k1_event_end(ctx, ev); };
  if (plan.tc) {
    if (tcsym) {
      const int npad = std::max(n_rows_pad, n_cols_pad);
      vec::pack_rhs(ctx, V_dev, cols->n, 1, npad, 1, 1, vpack, done);
      prof_begin();
      tcsym_kernel(done);
      prof_end();
      vec::tcsym_epilogue(ctx, partial, colpart, r_ptr, r_rec, c_ptr, c_rec, n_rows, plan.root_scale,
                          noise, noise_v, out_dev, done);
      return;
    }
    // V packed per part (column segments [0, split) and [split, n_seg)), each
    // with its own column scales, exactly as the staged upload packs it
    const int s_split = tc_split();
    if (s_split < n_seg) {
      const int64_t r_split = std::min<int64_t>((int64_t)s_split * tiles_per_seg * 64, cols->n);
      vec::pack_rhs_tc(ctx, V_dev, r_split, t, s_split * tiles_per_seg, tb, 1, vtc, vscale, v_inexact, done);
      vec::pack_rhs_tc(ctx, V_dev + r_split * t, cols->n - r_split, t,
                       (int)ceil_div<int64_t>(cols->n - r_split, 64), tb, 1,
                       static_cast<char*>(vtc) + (size_t)s_split * tiles_per_seg * 2 * tb * 64 * 2, vscale + tb,
                       v_inexact, done);
    } else {
      vec::pack_rhs_tc(ctx, V_dev, cols->n, t, n_tiles, tb, n_pass, vtc, vscale, v_inexact, done);
    }
    LgpTcArgs a = plan.tca;
    a.v_inexact = v_inexact;
    a.vscale = vscale;
    a.a1 = fr;
    a.b1 = fc;
    a.r32 = r32;
    a.c32 = c32;
    a.v = vtc;
    a.partial = partial;
    a.done = done;
    a.n_rows_pad = n_rows_pad;
    a.n_rb = n_rb;
    a.n_seg = n_seg;
    a.n_pass = n_pass;
    a.tiles_per_seg = tiles_per_seg;
    a.n_tiles = n_tiles;
    a.seg_base = 0;
    a.seg_split = s_split;
    const int64_t grid = (int64_t)n_rb * n_seg * n_pass;
    if (grid > 0x7fffffff) throw Error(LGP_E_UNSUPPORTED, "problem too large for one launch");
    prof_begin();
    launch(ctx, mod->matvec, (unsigned)grid, 1, plan.tune.threads, plan.smem_bytes, &a);
    prof_end();
    vec::epilogue(ctx, partial, n_seg, n_pass, n_rows_pad, tb, n_rows, t, plan.root_scale, noise,
                  noise_v, out_dev, done);
    return;
  }
  vec::pack_rhs(ctx, V_dev, cols->n, t, n_cols_pad, tb, n_pass, vpack, done);
  if (sym) {
    LgpMatvecArgs a = plan.mv;
    a.fr = fr;
    a.fc = fc;
    a.v = vpack;
    a.partial = partial;
    a.colpart = colpart;
    a.units = units;
    a.n_units = n_units;
    a.done = done;
    a.n_rows_pad = n_rows_pad;
    a.n_cols_pad = n_cols_pad;
    a.n_rb = n_rb;
    a.n_tiles = n_tiles;
    a.n_pass = n_pass;
    prof_begin();
    void* params[] = {&a};
    LGP_CU_CHECK(drv::LaunchKernel(mod->matvec_sym, (unsigned)n_units, (unsigned)n_pass, 1,
                                   plan.tune.threads, 1, 1, (unsigned)smem_sym,
                                   (CUstream)ctx->stream, params, nullptr));
    ++ctx->launches;
    prof_end();
    vec::sym_epilogue(ctx, partial, colpart, n_rb, plan.tune.threads * plan.tune.r, n_pass, tb,
                      n_rows, t, plan.root_scale, noise, noise_v, out_dev, done);
    return;
  }
  LgpMatvecArgs a = plan.mv;
  a.fr = fr;
  a.fc = fc;
  a.v = vpack;
  a.partial = partial;
  a.done = done;
  a.n_rows_pad = n_rows_pad;
  a.n_cols_pad = n_cols_pad;
  a.n_rb = n_rb;
  a.n_seg = n_seg;
  a.n_pass = n_pass;
  a.tiles_per_seg = tiles_per_seg;
  a.n_tiles = n_tiles;
  const int64_t grid = (int64_t)n_rb * n_seg * n_pass;
  if (grid > 0x7fffffff) throw Error(LGP_E_UNSUPPORTED, "problem too large for one launch");
  prof_begin();
  launch(ctx, mod->matvec, (unsigned)grid, 1, plan.tune.threads, plan.smem_bytes, &a);
  prof_end();
  vec::epilogue(ctx, partial, n_seg, n_pass, n_rows_pad, tb, n_rows, t, plan.root_scale, noise,
                noise_v, out_dev, done);
}

// ------------------------------------------------------------------ CG
DonePoller::DonePoller(Context* c, const int* d, int a) : ctx(c), done_dev(d), ahead(std::max(1, std::min(a, 15))) {
  if (!ctx->done_pin) LGP_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->done_pin), 16 * sizeof(int), 0));
  for (cudaEvent_t& e : ctx->done_ev)
    if (!e) LGP_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

bool DonePoller::check() {
  const int slot = tail % 16;
  LGP_CUDA_CHECK(cudaMemcpyAsync(ctx->done_pin + slot, done_dev, sizeof(int), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  LGP_CUDA_CHECK(cudaEventRecord(ctx->done_ev[slot], ctx->stream));
  ++tail;
  if (ctx->sharded()) {
    // every rank must leave the loop after the same iteration (each one
    // issues a collective): wait for this sample, whose value is the
    // device state after this iteration - identical on every rank -
    // instead of the first completed sample, which depends on timing
    bool any = false;
    for (; head < tail; ++head) {
      LGP_CUDA_CHECK(cudaEventSynchronize(ctx->done_ev[head % 16]));
      if (head == tail - 1) any = ctx->done_pin[head % 16] != 0;
    }
    return any;
  }
  while (head < tail) {
    const int h = head % 16;
    if (tail - head > ahead) {
      LGP_CUDA_CHECK(cudaEventSynchronize(ctx->done_ev[h]));
    } else {
      const cudaError_t q = cudaEventQuery(ctx->done_ev[h]);
      if (q == cudaErrorNotReady) break;
      LGP_CUDA_CHECK(q);
    }
    ++head;
    if (ctx->done_pin[h]) return true;
  }
  return false;
}

bool DonePoller::drain() {
  bool any = false;
  for (; head < tail; ++head) {
    LGP_CUDA_CHECK(cudaEventSynchronize(ctx->done_ev[head % 16]));
    any = any || ctx->done_pin[head % 16] != 0;
  }
  return any;
}

struct CgBuffers {
  double *x, *r, *p, *ap, *part, *bb;
  vec::CgState s;
};

static CgBuffers cg_buffers(Context* ctx, int64_t n_alloc, int t, int nblk) {
  CgBuffers b;
  const size_t vb = (size_t)n_alloc * t * 8;
  b.x = (double*)ctx->scratch_get("cg.x", vb);
  b.r = (double*)ctx->scratch_get("cg.r", vb);
  b.p = (double*)ctx->scratch_get("cg.p", vb);
  b.ap = (double*)ctx->scratch_get("cg.ap", vb);
  b.part = (double*)ctx->scratch_get("cg.part", (size_t)nblk * t * 8);
  char* sc = (char*)ctx->scratch_get("cg.scal", (size_t)t * 8 * 8 + 64);
  double* d = (double*)sc;
  b.bb = d;
  b.s.rs = d + t;
  b.s.tol = d + 2 * t;
  b.s.step = d + 3 * t;
  b.s.beta = d + 4 * t;
  b.s.res = d + 5 * t;
  int* iv = (int*)(d + 6 * t);
  b.s.active = iv;
  b.s.iters = iv + t;
  b.s.status = iv + 2 * t;
  b.s.done = iv + 2 * t + 1;
  b.s.bad_col = iv + 2 * t + 2;
  return b;
}

// B_dev: n_alloc x t device buffer (rows >= n ignored). Results stay on the
// device in the returned buffers' x; iterations / residuals copied to host.
void cg_device(Context* ctx, const KernelHandle* k, const Points* pts, double noise,
               const double* B_dev, int t, double rel_tol, int max_iter, double** x_dev,
               int32_t* iters_out, double* res_out, const CgShifts* shifts) {
  const int64_t n = pts->n;
  int64_t r0 = 0, r1 = n;
  lgp_partition(n, ctx->world, ctx->rank, &r0, &r1);
  const int64_t S = ceil_div<int64_t>(n, ctx->world);
  const int64_t n_alloc = S * ctx->world;
  const int nblk = vec::reduce_blocks(n, t);
  CgBuffers b = cg_buffers(ctx, n_alloc, t, nblk);
  if (max_iter <= 0) max_iter = (int)std::min<int64_t>(n, 1000);

  MatvecOp op;
  op.ctx = ctx;
  op.k = k;
  op.rows = pts;
  op.cols = pts;
  op.row0 = r0;
  op.n_rows = r1 - r0;
  op.t = t;
  op.tag = "cg.mv";
  // t = 1 (the alpha solve): exactly symmetric kernels only (K1-TC-sym /
  // SIMT), CG counts its iterations. Multi-RHS CG (predictive variance, t = T
  // test points): the tensor-core K1 - its rounding-level asymmetry costs
  // iterations (~1.3x) but each costs 4.5x less than the SIMT kernel's t/16
  // passes (cfg4, T = 200: 47 vs 210 ms).
  op.allow_tc = t >= 8;
  if (ctx->sharded() && t == 1 && !std::getenv("LGP_NO_RANK_SPLIT")) {
    // try the rank-split symmetric schedule: all rows, a share of the pairs
    op.rank_split = true;
    op.row0 = 0;
    op.n_rows = n;
    op.prepare();
    if (!op.tcsym) {  // ineligible tree: back to local rows + all-gather
      op = MatvecOp{};
      op.ctx = ctx;
      op.k = k;
      op.rows = pts;
      op.cols = pts;
      op.row0 = r0;
      op.n_rows = r1 - r0;
      op.t = t;
      op.tag = "cg.mv";
      op.prepare();
    }
  } else {
    op.prepare();
  }
  const bool split = op.rank_split && op.tcsym;
  // multi-pass multi-RHS CG on one rank: drop converged columns from the K1
  // passes as they converge (LGP_CG_NO_COMPACT=1 keeps every column)
  const bool compact = !ctx->sharded() && t > 1 && op.plan.tc && t > op.plan.tc_n &&
                       !std::getenv("LGP_CG_NO_COMPACT");
  int t_run = t;
  MatvecOp opc;
  int* cmap = nullptr;
  double *pc = nullptr, *apc = nullptr;
  if (compact) {
    cmap = (int*)ctx->scratch_get("cg.cmap", (size_t)t * sizeof(int));
    pc = (double*)ctx->scratch_get("cg.pc", (size_t)n_alloc * t * 8);
    apc = (double*)ctx->scratch_get("cg.apc", (size_t)n_alloc * t * 8);
  }

  vec::dot_partial(ctx, B_dev, B_dev, n, t, b.part, nullptr);
  vec::dot_final(ctx, b.part, nblk, t, b.bb, nullptr);
  vec::cg_init(ctx, B_dev, b.x, b.r, b.p, n, t, rel_tol, b.bb, b.s);
  // shifted systems on the seed's Krylov space (t = 1): two vectors each
  const int nsh = shifts ? shifts->n : 0;
  double *xs = nullptr, *ps = nullptr, *sig = nullptr;
  vec::CgShiftState* sst = nullptr;
  if (nsh > 0) {
    if (t != 1 || nsh > vec::kMaxShifts) throw Error(LGP_E_ARG, "shifted CG: one right-hand side, <= 64 shifts");
    ps = (double*)ctx->scratch_get("cg.sh.p", (size_t)n_alloc * nsh * 8);
    sig = (double*)ctx->scratch_get("cg.sh.sig", (size_t)nsh * 8);
    sst = (vec::CgShiftState*)ctx->scratch_get("cg.sh.state", 2 * sizeof(vec::CgShiftState));
    xs = shifts->xs_dev;
    LGP_CUDA_CHECK(cudaMemcpyAsync(sig, shifts->sig, (size_t)nsh * 8, cudaMemcpyHostToDevice, ctx->stream));
    vec::cg_shift_init(ctx, B_dev, n, nsh, xs, ps, sst);
  }

  // host-side stop checks: every iteration for large operators, else in
  // batches (kernels after convergence early-exit on the device flag)
  const double entries = (double)n * (double)n * t;
  // the host samples the device done flag every few iterations through
  // asynchronous copies (DonePoller): it never waits for the GPU to drain
  // (a synchronous check every 4 iterations left it idle ~30 us each time),
  // and iterations enqueued past convergence exit at their first instruction
  // (multi-rank: synchronous samples, so every 8 iterations - the few
  // iterations queued past convergence are no-ops on the device)
  int check_every = entries > 2e8 && !ctx->sharded() ? 2 : 8;
  if (const char* e = std::getenv("LGP_CG_CHECK")) check_every = std::max(1, atoi(e));
  DonePoller poll(ctx, b.s.done, entries > 2e8 ? 2 : 4);
  int done_h = 0;
  LGP_CUDA_CHECK(cudaMemcpyAsync(&done_h, b.s.done, sizeof(int), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  // single RHS on the symmetric tensor-core kernel: the fused iteration (4
  // launches: pack+p-update, K1, records+p.Ap+step, x/r update+r.r+beta)
  const bool fused = op.tcsym && t == 1 && !std::getenv("LGP_CG_UNFUSED");
  // one rank: the whole vector step is one cooperative launch (cg1_vec), the
  // next direction and K1 operand included (LGP_CG_VEC3=1: the 3-launch form)
  const bool vec1 = fused && !split && !std::getenv("LGP_CG_VEC3") && vec::cg1_vec_supported(ctx, n);
  // multi-rank: after the all-reduce of Ap, the same one-launch step from Ap
  // (p.Ap shares as k_cg1_pap's, then update, beta and the next direction)
  const bool vec1s = fused && split && !std::getenv("LGP_CG_VEC3") && vec::cg1_vec_supported(ctx, n);
  const int64_t n_pack = std::max(op.n_rows_pad, op.n_cols_pad);
  double *part1 = nullptr, *part2 = nullptr;
  unsigned* cnt1 = nullptr;
  if (fused) {
    const size_t np = (size_t)std::max<int64_t>(op.n_tiles, vec::cg1_blocks(n));
    const size_t ncnt = 4;  // the 3-launch form's ticket, or cg1_vec's barrier
    part1 = (double*)ctx->scratch_get("cg.part1", 2 * np * 8 + ncnt * 4);
    part2 = part1 + np;
    cnt1 = reinterpret_cast<unsigned*>(part1 + 2 * np);
    LGP_CUDA_CHECK(cudaMemsetAsync(cnt1, 0, ncnt * 4, ctx->stream));
    if (vec1 || vec1s) vec::cg1_pack(ctx, b.p, b.r, op.vpack, n, n_pack, b.s);  // beta = 0: p = r = b
  }
  unsigned long long* vtrace = nullptr;
  if (vec1 && std::getenv("LGP_CG_VEC_TRACE")) {
    vtrace = (unsigned long long*)ctx->scratch_get("cg.vtrace", (size_t)ctx->sm_count * 8 * 8);
    LGP_CUDA_CHECK(cudaMemsetAsync(vtrace, 0, (size_t)ctx->sm_count * 8 * 8, ctx->stream));
  }
  for (int it = 1; it <= max_iter && !done_h; ++it) {
    if (vec1) {
      {
        auto ev = k1_event_begin(ctx);
        op.tcsym_kernel(b.s.done);
        k1_event_end(ctx, ev);
      }
      vec::cg1_vec(ctx, op.partial, op.colpart, op.r_ptr, op.r_rec, op.c_ptr, op.c_rec, n, n_pack,
                   op.plan.root_scale, noise, b.x, b.r, b.p, b.ap, op.vpack, part1, part2, cnt1, it,
                   max_iter, b.s, vtrace);
      if (vtrace != nullptr && it == 3) {
        // diagnostics: phase boundaries of the third vector step, CTA 0 and
        // the latest CTA, microseconds from CTA 0's start
        std::vector<unsigned long long> tr((size_t)ctx->sm_count * 8);
        LGP_CUDA_CHECK(cudaMemcpyAsync(tr.data(), vtrace, tr.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
        LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        for (int k = 0; k < 8; ++k) {
          unsigned long long mx = 0;
          for (int bk = 0; bk < ctx->sm_count; ++bk) mx = std::max(mx, tr[(size_t)bk * 8 + k]);
          std::fprintf(stderr, "cg1_vec phase %d: cta0 %.2f us, max %.2f us\n", k, (tr[k] - tr[0]) * 1e-3,
                       (mx - tr[0]) * 1e-3);
        }
      }
      if (nsh > 0) vec::cg_shift(ctx, xs, ps, b.r, n, nsh, sig, sst, b.s, it);
    } else if (vec1s) {
      {
        auto ev = k1_event_begin(ctx);
        op.tcsym_kernel(b.s.done);
        k1_event_end(ctx, ev);
      }
      vec::tcsym_epilogue(ctx, op.partial, op.colpart, op.r_ptr, op.r_rec, op.c_ptr, op.c_rec, n,
                          op.plan.root_scale, ctx->rank == 0 ? noise : 0.0,
                          ctx->rank == 0 ? b.p : nullptr, b.ap, b.s.done);
      comm_allreduce_sum_inplace(ctx->comm, b.ap, (size_t)n, ctx->stream);
      vec::cg1_vec(ctx, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, n, n_pack, 1.0, 0.0, b.x,
                   b.r, b.p, b.ap, op.vpack, part1, part2, cnt1, it, max_iter, b.s, vtrace);
      if (nsh > 0) vec::cg_shift(ctx, xs, ps, b.r, n, nsh, sig, sst, b.s, it);
    } else if (fused) {
      vec::cg1_pack(ctx, b.p, b.r, op.vpack, n, n_pack, b.s);
      {
        auto ev = k1_event_begin(ctx);
        op.tcsym_kernel(b.s.done);
        k1_event_end(ctx, ev);
      }
      if (split) {
        vec::tcsym_epilogue(ctx, op.partial, op.colpart, op.r_ptr, op.r_rec, op.c_ptr, op.c_rec, n,
                            op.plan.root_scale, ctx->rank == 0 ? noise : 0.0,
                            ctx->rank == 0 ? b.p : nullptr, b.ap, b.s.done);
        comm_allreduce_sum_inplace(ctx->comm, b.ap, (size_t)n, ctx->stream);
        vec::cg1_pap(ctx, b.p, b.ap, n, part1, cnt1, b.s);
      } else {
        vec::tcsym_epilogue_cg(ctx, op.partial, op.colpart, op.r_ptr, op.r_rec, op.c_ptr, op.c_rec, n,
                               op.plan.root_scale, noise, b.p, b.ap, part1, cnt1, b.s);
      }
      vec::cg1_update(ctx, b.x, b.r, b.p, b.ap, n, part1, cnt1, it, max_iter, b.s);
      if (nsh > 0) vec::cg_shift(ctx, xs, ps, b.r, n, nsh, sig, sst, b.s, it);
    } else {
      if (split) {
        // this rank's pair share over all rows (noise term on rank 0 only), then
        // the sum over ranks: one all-reduce of n doubles per iteration
        op.run(b.p, b.ap, ctx->rank == 0 ? noise : 0.0, ctx->rank == 0 ? b.p : nullptr, b.s.done);
        comm_allreduce_sum_inplace(ctx->comm, b.ap, (size_t)n, ctx->stream);
      } else if (t_run < t) {
        // the still-active columns only (see the compaction below)
        vec::gather_cols(ctx, b.p, n, t, cmap, t_run, pc, b.s.done);
        opc.run(pc, apc, noise, pc, b.s.done);
        vec::scatter_cols(ctx, apc, n, t_run, cmap, t, b.ap, b.s.done);
      } else {
        op.run(b.p, b.ap + r0 * t, noise, b.p + r0 * t, b.s.done);
        if (ctx->sharded()) comm_allgather_inplace(ctx->comm, b.ap, (size_t)S * t, ctx->stream);
      }
      vec::dot_partial(ctx, b.p, b.ap, n, t, b.part, b.s.done);
      vec::cg_fin_pap(ctx, b.part, nblk, t, b.s);
      vec::cg_update_xr(ctx, b.x, b.r, b.p, b.ap, n, t, b.s, b.part);
      vec::cg_fin_rs(ctx, b.part, nblk, t, it, max_iter, b.s);
      if (nsh > 0) vec::cg_shift(ctx, xs, ps, b.r, n, nsh, sig, sst, b.s, it);
      vec::cg_update_p(ctx, b.p, b.r, n, t, b.s);
    }
    if (it % check_every == 0 || it == max_iter) done_h = poll.check();
    if (compact && it % 8 == 0 && !done_h) {
      // columns converge at different iterations (cfg4 predictive variance:
      // 608-804): once the active ones fit in fewer K1 passes, run only those
      // (converged columns are never updated again, so a mask read a few
      // iterations late is a superset of the active set)
      std::vector<int> act(t);
      LGP_CUDA_CHECK(cudaMemcpyAsync(act.data(), b.s.active, t * sizeof(int), cudaMemcpyDeviceToHost,
                                     ctx->stream));
      LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
      std::vector<int> cols;
      for (int c = 0; c < t; ++c)
        if (act[c]) cols.push_back(c);
      const int tb = op.plan.tc_n;
      if (!cols.empty() && ceil_div<int>((int)cols.size(), tb) < ceil_div<int>(t_run, tb)) {
        t_run = (int)cols.size();
        LGP_CUDA_CHECK(cudaMemcpyAsync(cmap, cols.data(), cols.size() * sizeof(int),
                                       cudaMemcpyHostToDevice, ctx->stream));
        opc = MatvecOp{};
        opc.ctx = ctx;
        opc.k = k;
        opc.rows = pts;
        opc.cols = pts;
        opc.row0 = 0;
        opc.n_rows = n;
        opc.t = t_run;
        // the same RHS-per-pass kernel and column segments: per-column results
        // bit-identical to the full pass set
        opc.tc_t_hint = t;
        opc.tiles_per_seg_hint = op.tiles_per_seg;
        opc.allow_tc = true;
        opc.tag = "cg.mvc";
        opc.prepare();
      }
    }
  }
  poll.drain();
  int status[2] = {0, -1};
  LGP_CUDA_CHECK(cudaMemcpyAsync(status, b.s.status, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  LGP_CUDA_CHECK(cudaMemcpyAsync(iters_out, b.s.iters, t * sizeof(int), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  LGP_CUDA_CHECK(cudaMemcpyAsync(res_out, b.s.res, t * sizeof(double), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  if (nsh > 0) {
    // the state the iteration after the seed's last one would read
    int last = 0;
    LGP_CUDA_CHECK(cudaMemcpyAsync(&last, b.s.iters, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    const vec::CgShiftState* fin = sst + ((last + 1) & 1);
    LGP_CUDA_CHECK(cudaMemcpyAsync(shifts->iters, fin->iters, nsh * sizeof(int), cudaMemcpyDeviceToHost,
                                   ctx->stream));
    LGP_CUDA_CHECK(cudaMemcpyAsync(shifts->res, fin->res, nsh * sizeof(double), cudaMemcpyDeviceToHost,
                                   ctx->stream));
  }
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  if (status[0] != 0)
    throw Error(LGP_E_NOT_SPD, "CG breakdown: p.A.p is not positive (column " +
                                   std::to_string(status[1]) + ")");
  *x_dev = b.x;
}

// ------------------------------------------------------------- Lanczos
void lanczos_device(Context* ctx, const KernelHandle* k, const Points* pts, double noise,
                    const double* Z_dev, int t, int steps, double* alphas, double* betas,
                    int32_t* steps_out) {
  const int64_t n = pts->n;
  int64_t r0 = 0, r1 = n;
  lgp_partition(n, ctx->world, ctx->rank, &r0, &r1);
  const int64_t S = ceil_div<int64_t>(n, ctx->world);
  const int64_t n_alloc = S * ctx->world;
  const int nblk = vec::reduce_blocks(n, t);
  const size_t vb = (size_t)n_alloc * t;
  double* basis = (double*)ctx->scratch_get("lz.basis", vb * steps * 8);
  double* w = (double*)ctx->scratch_get("lz.w", vb * 8);
  double* part = (double*)ctx->scratch_get("lz.part", (size_t)nblk * steps * t * 8);
  char* sc = (char*)ctx->scratch_get("lz.scal", (size_t)t * 8 * (2 * steps + steps + 4) + 64);
  double* d = (double*)sc;
  vec::LzState s;
  s.alpha = d;
  s.beta = d + (size_t)t * steps;
  s.h = d + (size_t)2 * t * steps;
  s.a_cur = s.h + (size_t)t * steps;
  s.nrm = s.a_cur + t;
  double* zz = s.nrm + t;
  int* iv = (int*)(zz + t);
  s.active = iv;
  s.count = iv + t;
  s.done = iv + 2 * t;
  LGP_CUDA_CHECK(cudaMemsetAsync(s.alpha, 0, (size_t)2 * t * steps * 8, ctx->stream));

  MatvecOp op;
  op.ctx = ctx;
  op.k = k;
  op.rows = pts;
  op.cols = pts;
  op.row0 = r0;
  op.n_rows = r1 - r0;
  op.t = t;
  op.allow_tc = true;
  op.tag = "lz.mv";
  op.prepare();

  vec::dot_partial(ctx, Z_dev, Z_dev, n, t, part, nullptr);
  vec::dot_final(ctx, part, nblk, t, zz, nullptr);
  vec::lz_init(ctx, Z_dev, basis, n, t, zz, s);
  const int64_t stride = (int64_t)n_alloc * t;
  const double entries = (double)n * (double)n * t;
  // the host samples the device done flag every few iterations through
  // asynchronous copies (DonePoller): it never waits for the GPU to drain
  // (a synchronous check every 4 iterations left it idle ~30 us each time),
  // and iterations enqueued past convergence exit at their first instruction
  // (multi-rank: synchronous samples, so every 8 iterations - the few
  // iterations queued past convergence are no-ops on the device)
  int check_every = entries > 2e8 && !ctx->sharded() ? 2 : 8;
  if (const char* e = std::getenv("LGP_CG_CHECK")) check_every = std::max(1, atoi(e));
  DonePoller poll(ctx, s.done, entries > 2e8 ? 2 : 4);
  int done_h = 0;
  for (int j = 0; j < steps && !done_h; ++j) {
    double* q = basis + (size_t)j * stride;
    const double* qprev = j > 0 ? basis + (size_t)(j - 1) * stride : nullptr;
    op.run(q, w + r0 * t, noise, q + r0 * t, s.done);
    if (ctx->sharded()) comm_allgather_inplace(ctx->comm, w, (size_t)S * t, ctx->stream);
    vec::dot_partial(ctx, q, w, n, t, part, s.done);
    vec::lz_fin_alpha(ctx, part, nblk, t, j, steps, s);
    vec::lz_update1(ctx, w, q, qprev, n, t, j, steps, s);
    if (j == steps - 1) break;  // the last step needs no beta (solvers.py:148-149)
    vec::lz_multidot(ctx, basis, stride, j + 1, w, n, t, part, s.done);
    vec::lz_fin_h(ctx, part, nblk, j + 1, t, s);
    vec::lz_update2(ctx, w, basis, stride, j + 1, n, t, s, part);
    vec::lz_fin_beta(ctx, part, nblk, t, j, steps, s);
    vec::lz_normalize(ctx, w, basis + (size_t)(j + 1) * stride, n, t, s);
    if ((j + 1) % check_every == 0) done_h = poll.check();
  }
  poll.drain();
  std::vector<double> al((size_t)t * steps), be((size_t)t * steps);
  LGP_CUDA_CHECK(cudaMemcpyAsync(al.data(), s.alpha, al.size() * 8, cudaMemcpyDeviceToHost,
                                 ctx->stream));
  LGP_CUDA_CHECK(cudaMemcpyAsync(be.data(), s.beta, be.size() * 8, cudaMemcpyDeviceToHost,
                                 ctx->stream));
  LGP_CUDA_CHECK(cudaMemcpyAsync(steps_out, s.count, t * sizeof(int), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  for (int c = 0; c < t; ++c) {
    for (int j = 0; j < steps; ++j) alphas[(size_t)c * steps + j] = al[(size_t)c * steps + j];
    for (int j = 0; j + 1 < steps; ++j)
      betas[(size_t)c * (steps - 1) + j] = be[(size_t)c * steps + j];
  }
}

}  // namespace lgp

// C ABI front end (include/lightgp.h): argument validation with the
// reference's error taxonomy, host<->device staging, and dispatch into the
// matvec engine and solver drivers. Every entry point is exception-safe and
// returns a status code; the message is kept per thread.
#include <cmath>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "lgp_internal.h"

using namespace lgp;

namespace lgp {
static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace lgp

struct lgp_ctx : Context {};

namespace {
// Live contexts: objects that outlive their context (point sets freed by a
// garbage collector after the context) must not touch it.
std::mutex g_ctx_mu;
std::set<const Context*> g_live;
bool ctx_alive(const Context* c) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  return g_live.count(c) != 0;
}
}  // namespace
struct lgp_kernel : KernelHandle {};
struct lgp_points : Points {};

#define API_BEGIN try {
#define API_END                               \
  }                                           \
  catch (const Error& e) {                    \
    set_last_error(e.what());                 \
    return e.code;                            \
  }                                           \
  catch (const std::bad_alloc&) {             \
    set_last_error("host allocation failed"); \
    return LGP_E_OOM;                         \
  }                                           \
  catch (const std::exception& e) {           \
    set_last_error(e.what());                 \
    return LGP_E_CUDA;                        \
  }                                           \
  return LGP_OK;

namespace {

void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

// Multithreaded finiteness scan (up to 8 threads, >= 2 MB each): a double is
// finite iff its exponent field is not all ones; (u & m) + 2^52 carries into
// bit 63 exactly then. Adds and ORs vectorise with baseline SSE2.
bool all_finite_mt(const double* p, size_t n) {
  auto scan = [p](size_t lo, size_t hi) {
    const uint64_t* u = reinterpret_cast<const uint64_t*>(p);
    const uint64_t m = 0x7ff0000000000000ull;
    uint64_t acc = 0;
    for (size_t i = lo; i < hi; ++i) acc |= (u[i] & m) + (uint64_t(1) << 52);
    return (acc >> 63) != 0;
  };
  const size_t kPerThread = size_t(1) << 18;
  unsigned nt = std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency()));
  nt = (unsigned)std::min<size_t>(nt, (n + kPerThread - 1) / kPerThread);
  if (nt <= 1) return !scan(0, n);
  std::vector<char> flags(nt, 0);
  std::vector<std::thread> th;
  const size_t step = (n + nt - 1) / nt;
  for (unsigned k = 1; k < nt; ++k)
    th.emplace_back([&, k] { flags[k] = scan(std::min(n, k * step), std::min(n, (k + 1) * step)); });
  flags[0] = scan(0, std::min(n, step));
  for (auto& x : th) x.join();
  for (char f : flags)
    if (f) return false;
  return true;
}

void check_finite(const double* p, size_t n, const char* name) {
  if (!all_finite_mt(p, n))
    throw Error(LGP_E_NONFINITE, std::string(name) + " contains NaN or infinite entries");
}

// Stage a host or device input (n x t) into a device buffer of n_alloc rows.
const double* stage_in(Context* ctx, const char* name, const double* src, int64_t n, int t,
                       int64_t n_alloc, uint32_t flags) {
  const size_t bytes = (size_t)n * t * 8;
  if ((flags & LGP_DEVICE_PTRS) && n_alloc == n) return src;
  double* d = (double*)ctx->scratch_get(name, (size_t)n_alloc * t * 8);
  if (n_alloc > n)
    LGP_CUDA_CHECK(cudaMemsetAsync(d + (size_t)n * t, 0, (size_t)(n_alloc - n) * t * 8, ctx->stream));
  LGP_CUDA_CHECK(cudaMemcpyAsync(d, src, bytes,
                                 (flags & LGP_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice
                                                           : cudaMemcpyHostToDevice,
                                 ctx->stream));
  return d;
}

void stage_out(Context* ctx, double* dst, const double* src, size_t bytes, uint32_t flags) {
  if (dst == src) return;
  LGP_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes,
                                 (flags & LGP_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice
                                                           : cudaMemcpyDeviceToHost,
                                 ctx->stream));
}

Plan plan_for(const KernelHandle* k, int d) { return make_plan(k->tree, d, 1, 0); }

}  // namespace

extern "C" {

int lgp_abi_version(void) { return LGP_ABI_VERSION; }

const char* lgp_last_error(void) { return g_last_error.c_str(); }

int lgp_device_count(int* out) {
  API_BEGIN
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *out = n;
  API_END
}

int lgp_partition(int64_t n, int world, int rank, int64_t* r0, int64_t* r1) {
  API_BEGIN
  require(n >= 0 && world >= 1 && rank >= 0 && rank < world, LGP_E_ARG, "bad partition request");
  const int64_t s = (n + world - 1) / world;
  int64_t a = (int64_t)rank * s, b = a + s;
  if (a > n) a = n;
  if (b > n) b = n;
  *r0 = a;
  *r1 = b;
  API_END
}

int lgp_comm_unique_id(uint8_t* out128) {
  API_BEGIN
  comm_unique_id(out128);
  API_END
}

int lgp_comm_allreduce_max(lgp_ctx* ctx, double* vals, int32_t count) {
  API_BEGIN
  require(ctx != nullptr && (vals != nullptr || count == 0) && count >= 0, LGP_E_ARG,
          "bad all-reduce request");
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  if (ctx->comm) comm_allreduce_max_host(ctx->comm, vals, count, ctx->stream);
  API_END
}

int lgp_ctx_create(int device, int rank, int world, const uint8_t* nccl_id, lgp_ctx** out) {
  API_BEGIN
  require(out != nullptr, LGP_E_ARG, "out is null");
  require(world >= 1 && rank >= 0 && rank < world, LGP_E_ARG, "bad rank / world");
  require(world == 1 || nccl_id != nullptr, LGP_E_ARG, "multi-rank context needs an NCCL id");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw Error(LGP_E_CUDA, "no CUDA device available (the lightgp hot path has no CPU fallback)");
  }
  require(device >= 0 && device < ndev, LGP_E_ARG, "device index out of range");
  std::unique_ptr<lgp_ctx> c(new lgp_ctx);
  c->device = device;
  c->rank = rank;
  c->world = world;
  c->activate();
  LGP_CUDA_CHECK(cudaFree(nullptr));  // create / retain the primary context
  int major = 0;
  LGP_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  require(major == 10, LGP_E_UNSUPPORTED, "this build targets sm_100a (B200) only");
  LGP_CUDA_CHECK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
  LGP_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  LGP_CUDA_CHECK(cudaEventCreate(&c->ev0));
  LGP_CUDA_CHECK(cudaEventCreate(&c->ev1));
  if (world > 1 || nccl_id != nullptr) c->comm = comm_create(rank, world, nccl_id, c->stream);
  {
    std::lock_guard<std::mutex> g(g_ctx_mu);
    g_live.insert(c.get());
  }
  *out = c.release();
  API_END
}

int lgp_ctx_destroy(lgp_ctx* ctx) {
  API_BEGIN
  if (!ctx) return LGP_OK;
  {
    std::lock_guard<std::mutex> g(g_ctx_mu);
    if (!g_live.erase(ctx)) return LGP_OK;  // idempotent
  }
  ctx->activate();
  cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->scratch)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  for (auto& kv : ctx->modules)
    if (kv.second->mod) drv::ModuleUnload(kv.second->mod);
  if (ctx->flush_buf) cudaFree(ctx->flush_buf);
  if (ctx->done_pin) cudaFreeHost(ctx->done_pin);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  for (cudaEvent_t e : ctx->copy_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->done_ev)
    if (e) cudaEventDestroy(e);
  for (auto& kv : ctx->pool)
    for (void* q : kv.second) cudaFree(q);
  for (auto& ev : ctx->ev_pending) ctx->ev_pool.push_back(ev);
  for (auto& ev : ctx->ev_pool) {
    cudaEventDestroy(ev.first);
    cudaEventDestroy(ev.second);
  }
  comm_destroy(ctx->comm);
  cudaEventDestroy(ctx->ev0);
  cudaEventDestroy(ctx->ev1);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  API_END
}

int lgp_ctx_sync(lgp_ctx* ctx) {
  API_BEGIN
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  API_END
}

int lgp_ctx_launch_count(lgp_ctx* ctx, uint64_t* out) {
  API_BEGIN
  *out = ctx->launches;
  API_END
}

int lgp_ctx_set_profile(lgp_ctx* ctx, int on) {
  API_BEGIN
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->profile = on != 0;
  API_END
}

int lgp_ctx_profile(lgp_ctx* ctx, double* k1_ms_total, uint64_t* k1_launches, int reset) {
  API_BEGIN
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  for (auto& ev : ctx->ev_pending) {
    float ms = 0.f;
    LGP_CUDA_CHECK(cudaEventElapsedTime(&ms, ev.first, ev.second));
    ctx->prof_ms += ms;
    ctx->prof_count += 1;
    ctx->ev_pool.push_back(ev);
  }
  ctx->ev_pending.clear();
  if (k1_ms_total) *k1_ms_total = ctx->prof_ms;
  if (k1_launches) *k1_launches = ctx->prof_count;
  if (reset) {
    ctx->prof_ms = 0.0;
    ctx->prof_count = 0;
  }
  API_END
}

int lgp_timer_start(lgp_ctx* ctx) {
  API_BEGIN
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  LGP_CUDA_CHECK(cudaEventRecord(ctx->ev0, ctx->stream));
  API_END
}

int lgp_timer_stop(lgp_ctx* ctx, float* ms) {
  API_BEGIN
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  LGP_CUDA_CHECK(cudaEventRecord(ctx->ev1, ctx->stream));
  LGP_CUDA_CHECK(cudaEventSynchronize(ctx->ev1));
  LGP_CUDA_CHECK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
  API_END
}

int lgp_device_alloc(lgp_ctx* ctx, size_t bytes, void** out) {
  API_BEGIN
  ctx->activate();
  LGP_CUDA_CHECK(cudaMalloc(out, bytes ? bytes : 16));
  API_END
}

int lgp_device_free(lgp_ctx* ctx, void* ptr) {
  API_BEGIN
  ctx->activate();
  if (ptr) LGP_CUDA_CHECK(cudaFree(ptr));
  API_END
}

int lgp_memcpy_h2d(lgp_ctx* ctx, void* dst, const void* src, size_t bytes) {
  API_BEGIN
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  LGP_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  API_END
}

int lgp_memcpy_d2h(lgp_ctx* ctx, void* dst, const void* src, size_t bytes) {
  API_BEGIN
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  LGP_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  API_END
}

int lgp_all_finite(const double* p, size_t n, int* all_finite) {
  API_BEGIN
  require(all_finite && (n == 0 || p), LGP_E_ARG, "bad lgp_all_finite arguments");
  *all_finite = all_finite_mt(p, n) ? 1 : 0;
  API_END
}

int lgp_host_alloc(size_t bytes, void** out) {
  API_BEGIN
  LGP_CUDA_CHECK(cudaMallocHost(out, bytes ? bytes : 16));
  API_END
}

int lgp_host_free(void* ptr) {
  API_BEGIN
  if (ptr) LGP_CUDA_CHECK(cudaFreeHost(ptr));
  API_END
}

int lgp_flush_l2(lgp_ctx* ctx, size_t bytes) {
  API_BEGIN
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  if (ctx->flush_bytes < bytes) {
    if (ctx->flush_buf) LGP_CUDA_CHECK(cudaFree(ctx->flush_buf));
    LGP_CUDA_CHECK(cudaMalloc(&ctx->flush_buf, bytes));
    ctx->flush_bytes = bytes;
  }
  LGP_CUDA_CHECK(cudaMemsetAsync(ctx->flush_buf, ctx->launches & 0xff, bytes, ctx->stream));
  API_END
}

// ------------------------------------------------------------ kernel trees
int lgp_kernel_compile(lgp_ctx* ctx, int n_nodes, const int32_t* kinds, const double* params,
                       int n_params, lgp_kernel** out) {
  API_BEGIN
  require(out && kinds && n_nodes >= 1, LGP_E_ARG, "bad kernel tree arguments");
  std::unique_ptr<lgp_kernel> k(new lgp_kernel);
  k->ctx = ctx;
  int need = 1, pi = 0;
  for (int i = 0; i < n_nodes; ++i) {
    const int kind = kinds[i];
    require(kind >= LGP_NODE_RBF && kind <= LGP_NODE_PRODUCT, LGP_E_ARG, "unknown node kind");
    require(need > 0, LGP_E_ARG, "kernel tree has trailing nodes");
    need += node_arity(kind) - 1;
    Node nd{kind, {0.0, 0.0}};
    const int np = node_nparams(kind);
    for (int q = 0; q < np; ++q) {
      require(pi < n_params && params, LGP_E_ARG, "too few kernel parameters");
      const double v = params[pi++];
      require(std::isfinite(v) && v > 0.0, LGP_E_ARG, "kernel parameters must be positive and finite");
      nd.p[q] = v;
    }
    k->tree.nodes.push_back(nd);
  }
  require(need == 0, LGP_E_ARG, "kernel tree is incomplete");
  require(pi == n_params, LGP_E_ARG, "too many kernel parameters");
  *out = k.release();
  API_END
}

int lgp_kernel_jit(const lgp_kernel* k, int32_t d, int32_t t, uint32_t flags, char* log,
                   size_t cap) {
  API_BEGIN
  require(k && d >= 1 && t >= 1, LGP_E_ARG, "bad arguments");
  int tb = 1;
  while (tb < t && tb < 16) tb <<= 1;
  Plan p = make_plan(k->tree, d, tb, flags);
  std::string lg;
  jit_compile(p.source, &lg);
  Plan tp = make_tc_plan(k->tree, d, t, flags);
  if (tp.tc) {
    std::string lg2;
    jit_compile(tp.source, &lg2);
    lg += "\n[tensor-core module]\n" + lg2;
  }
  if (log && cap) {
    const size_t n = std::min(cap - 1, lg.size());
    std::memcpy(log, lg.data(), n);
    log[n] = 0;
  }
  API_END
}

int lgp_kernel_free(lgp_kernel* k) {
  API_BEGIN
  delete k;
  API_END
}

int lgp_kernel_source(const lgp_kernel* k, int32_t d, int32_t t, uint32_t flags, char* buf,
                      size_t cap, size_t* needed) {
  API_BEGIN
  require(k && d >= 1 && t >= 1, LGP_E_ARG, "bad arguments");
  int tb = 1;
  while (tb < t && tb < 16) tb <<= 1;
  Plan p = make_tc_plan(k->tree, d, t, flags);
  if (!p.tc) p = make_plan(k->tree, d, tb, flags);
  if (needed) *needed = p.source.size() + 1;
  if (buf && cap) {
    const size_t n = std::min(cap - 1, p.source.size());
    std::memcpy(buf, p.source.data(), n);
    buf[n] = 0;
  }
  API_END
}

// -------------------------------------------------------------- point sets
int lgp_points_upload(lgp_ctx* ctx, const double* X, int64_t n, int32_t d, lgp_points** out) {
  API_BEGIN
  require(ctx && out, LGP_E_ARG, "bad points arguments");
  require(n >= 0 && d >= 1, LGP_E_DIM, "points must be n x d with d >= 1");
  require(n == 0 || X, LGP_E_ARG, "X is null");
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  std::unique_ptr<lgp_points> p(new lgp_points);
  p->ctx = ctx;
  p->n = n;
  p->d = d;
  const size_t xbytes = ((size_t)std::max<int64_t>(n, 1) * d * 8 + 255) / 256 * 256;
  p->bytes = xbytes + (size_t)d * 8;
  p->x = (double*)ctx->pool_get(p->bytes);
  p->ctr = (double*)((char*)p->x + xbytes);
  // finiteness, mean and radius are computed on the device right after the
  // copy (one pass over X in HBM instead of host scans of the caller's array)
  double* scratch = (double*)ctx->scratch_get(
      "pts.part", (size_t)vec::reduce_blocks(std::max<int64_t>(n, 1), 1) * d * 8);
  double* stats = (double*)ctx->scratch_get("pts.stats", (size_t)(d + 2) * 8);
  if (n > 0)
    LGP_CUDA_CHECK(cudaMemcpyAsync(p->x, X, (size_t)n * d * 8, cudaMemcpyHostToDevice, ctx->stream));
  vec::point_stats(ctx, p->x, n, d, p->ctr, scratch, stats);
  std::vector<double> h((size_t)d + 2);
  LGP_CUDA_CHECK(cudaMemcpyAsync(h.data(), stats, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));  // the host X may be freed after return
  int bad = 0;
  std::memcpy(&bad, &h[d + 1], sizeof(int));
  if (bad) {
    ctx->pool_put(p->x, p->bytes);
    throw Error(LGP_E_NONFINITE, "X contains NaN or infinite entries");
  }
  p->center.assign(h.begin(), h.begin() + d);
  p->radius = std::sqrt(h[d]);
  *out = p.release();
  API_END
}

int lgp_points_free(lgp_points* p) {
  API_BEGIN
  if (!p) return LGP_OK;
  if (ctx_alive(p->ctx)) {
    std::lock_guard<std::recursive_mutex> g(p->ctx->mu);
    // stream-ordered reuse: later work on the context stream may recycle it
    p->ctx->pool_put(p->x, p->bytes);
  }
  delete p;
  API_END
}

// ---------------------------------------------------------------- hot path
int lgp_matvec(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* rows, const lgp_points* cols,
               double noise, const double* V, int32_t t, double* out, uint32_t flags) {
  API_BEGIN
  require(ctx && k && rows && cols && out, LGP_E_ARG, "null argument");
  require(rows->d == cols->d, LGP_E_DIM, "row and column point sets differ in dimension");
  require(t >= 1, LGP_E_ARG, "t must be at least 1");
  require(std::isfinite(noise) && noise >= 0.0, LGP_E_ARG, "noise must be finite and nonnegative");
  require(cols->n == 0 || V, LGP_E_ARG, "V is null");
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  const bool square = (rows == cols);
  const int64_t n = rows->n;
  if (n == 0) return LGP_OK;
  int64_t r0 = 0, r1 = n;
  lgp_partition(n, ctx->world, ctx->rank, &r0, &r1);
  const int64_t S = (n + ctx->world - 1) / ctx->world;
  const int64_t n_alloc = S * ctx->world;
  const bool scan_v = !(flags & (LGP_DEVICE_PTRS | LGP_INPUTS_FINITE));
  double* od = (flags & LGP_DEVICE_PTRS) && !ctx->sharded()
                   ? out
                   : (double*)ctx->scratch_get("api.out", (size_t)n_alloc * t * 8);
  if (cols->n == 0) {
    if (scan_v) check_finite(V, (size_t)cols->n * t, "V");
    LGP_CUDA_CHECK(cudaMemsetAsync(od, 0, (size_t)n * t * 8, ctx->stream));
  } else {
    MatvecOp op;
    op.ctx = ctx;
    op.k = k;
    op.rows = rows;
    op.cols = cols;
    op.row0 = r0;
    op.n_rows = r1 - r0;
    op.t = t;
    op.flags = flags;
    op.allow_tc = true;
    op.flags |= kTcAnyT;
    op.tag = "api.mv";
    op.prepare();
    // host V on one GPU through the tensor-core kernel: the upload in two
    // parts, the second overlapping the first part's K1 (MatvecOp::run_staged)
    bool staged = false;
    if (!(flags & LGP_DEVICE_PTRS) && !ctx->sharded() && !std::getenv("LGP_NO_STAGED")) {
      double* vd = (double*)ctx->scratch_get("api.V", (size_t)cols->n * t * 8);
      staged = op.run_staged(V, vd, od, square ? noise : 0.0, square, [&]() {
        if (scan_v) check_finite(V, (size_t)cols->n * t, "V");  // while part 0's K1 runs
      });
    }
    if (!staged) {
      const double* Vd = stage_in(ctx, "api.V", V, cols->n, t, cols->n, flags);
      // validate V on the host while its copy is in flight (pinned V: the DMA
      // and the scan overlap); a non-finite V throws before any kernel is launched
      if (scan_v) check_finite(V, (size_t)cols->n * t, "V");
      op.run(Vd, od + r0 * t, square ? noise : 0.0, square ? Vd + r0 * t : nullptr, nullptr);
    }
    if (ctx->sharded()) comm_allgather_inplace(ctx->comm, od, (size_t)S * t, ctx->stream);
  }
  stage_out(ctx, out, od, (size_t)n * t * 8, flags);
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  API_END
}

int lgp_cg(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* pts, double noise, const double* B,
           int32_t t, double rel_tol, int32_t max_iter, double* X_out, int32_t* iters_out,
           double* final_res_out, uint32_t flags) {
  API_BEGIN
  require(ctx && k && pts && X_out && iters_out && final_res_out, LGP_E_ARG, "null argument");
  require(t >= 1 && t <= 256, LGP_E_ARG, "t must be in [1, 256]");
  require(rel_tol > 0.0, LGP_E_ARG, "rel_tolerance must be positive");
  require(std::isfinite(noise) && noise >= 0.0, LGP_E_ARG, "noise must be finite and nonnegative");
  const int64_t n = pts->n;
  require(n >= 1, LGP_E_DIM, "need at least one point");
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  const int64_t S = (n + ctx->world - 1) / ctx->world;
  const int64_t n_alloc = S * ctx->world;
  const double* Bd = stage_in(ctx, "api.B", B, n, t, n_alloc, flags);
  if (!(flags & (LGP_DEVICE_PTRS | LGP_INPUTS_FINITE))) check_finite(B, (size_t)n * t, "b");  // during the copy
  double* xd = nullptr;
  cg_device(ctx, k, pts, noise, Bd, t, rel_tol, max_iter, &xd, iters_out, final_res_out);
  stage_out(ctx, X_out, xd, (size_t)n * t * 8, flags);
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  API_END
}

int lgp_cg_shifted(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* pts, double noise,
                   const double* b, int32_t n_shifts, const double* shifts, double rel_tol,
                   int32_t max_iter, double* X_out, int32_t* iters_out, double* final_res_out,
                   uint32_t flags) {
  API_BEGIN
  require(ctx && k && pts && b && shifts && X_out && iters_out && final_res_out, LGP_E_ARG,
          "null argument");
  require(n_shifts >= 1 && n_shifts <= 64, LGP_E_ARG, "n_shifts must be in [1, 64]");
  require(rel_tol > 0.0, LGP_E_ARG, "rel_tolerance must be positive");
  require(std::isfinite(noise) && noise >= 0.0, LGP_E_ARG, "noise must be finite and nonnegative");
  for (int e = 0; e < n_shifts; ++e)
    require(std::isfinite(shifts[e]) && shifts[e] >= 0.0, LGP_E_ARG,
            "shifts must be finite and nonnegative (the seed has the smallest noise)");
  const int64_t n = pts->n;
  require(n >= 1, LGP_E_DIM, "need at least one point");
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  const int64_t S = (n + ctx->world - 1) / ctx->world;
  const int64_t n_alloc = S * ctx->world;
  const double* Bd = stage_in(ctx, "api.B", b, n, 1, n_alloc, flags);
  if (!(flags & (LGP_DEVICE_PTRS | LGP_INPUTS_FINITE))) check_finite(b, (size_t)n, "b");
  double* xs = (double*)ctx->scratch_get("api.Xs", (size_t)n_alloc * n_shifts * 8);
  CgShifts sh;
  sh.n = n_shifts;
  sh.sig = shifts;
  sh.xs_dev = xs;
  sh.iters = iters_out;
  sh.res = final_res_out;
  double* xd = nullptr;
  int32_t it_seed = 0;
  double res_seed = 0.0;
  cg_device(ctx, k, pts, noise, Bd, 1, rel_tol, max_iter, &xd, &it_seed, &res_seed, &sh);
  stage_out(ctx, X_out, xs, (size_t)n * n_shifts * 8, flags);
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  API_END
}

int lgp_lanczos(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* pts, double noise,
                const double* Z, int32_t t, int32_t steps, double* alphas, double* betas,
                int32_t* steps_out, uint32_t flags) {
  API_BEGIN
  require(ctx && k && pts && Z && alphas && betas && steps_out, LGP_E_ARG, "null argument");
  require(t >= 1 && t <= 256, LGP_E_ARG, "t must be in [1, 256]");
  require(steps >= 1, LGP_E_ARG, "lanczos_steps must be at least 1");
  const int64_t n = pts->n;
  require(n >= 1, LGP_E_DIM, "need at least one point");
  require(steps <= n, LGP_E_ARG, "steps must not exceed n");
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  const int64_t S = (n + ctx->world - 1) / ctx->world;
  const int64_t n_alloc = S * ctx->world;
  const double* Zd = stage_in(ctx, "api.Z", Z, n, t, n_alloc, flags);
  if (!(flags & (LGP_DEVICE_PTRS | LGP_INPUTS_FINITE))) check_finite(Z, (size_t)n * t, "z");  // during the copy
  lanczos_device(ctx, k, pts, noise, Zd, t, steps, alphas, betas, steps_out);
  API_END
}

int lgp_gram(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* rows, const lgp_points* cols,
             double* out, uint32_t flags) {
  API_BEGIN
  require(ctx && k && rows && cols && out, LGP_E_ARG, "null argument");
  require(rows->d == cols->d, LGP_E_DIM, "row and column point sets differ in dimension");
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  const size_t bytes = (size_t)rows->n * cols->n * 8;
  if (bytes == 0) return LGP_OK;
  Plan plan = plan_for(k, rows->d);
  Module* mod = get_module(ctx, plan);
  double* od = (flags & LGP_DEVICE_PTRS) ? out : (double*)ctx->scratch_get("api.gram", bytes);
  LgpGramArgs a = plan.gram;
  a.x = rows->x;
  a.y = cols->x;
  a.out = od;
  a.n_rows = rows->n;
  a.n_cols = cols->n;
  a.ld = cols->n;
  int64_t gy = (cols->n + 255) / 256;
  if (gy > 65535) gy = 65535;
  require(rows->n <= 0x7fffffff, LGP_E_UNSUPPORTED, "too many rows for one gram launch");
  void* params[] = {&a};
  LGP_CU_CHECK(drv::LaunchKernel(mod->gram, (unsigned)rows->n, (unsigned)gy, 1, 256, 1, 1, 0,
                              (CUstream)ctx->stream, params, nullptr));
  ++ctx->launches;
  stage_out(ctx, out, od, bytes, flags);
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  API_END
}

int lgp_diag(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* pts, double* out,
             uint32_t flags) {
  API_BEGIN
  require(ctx && k && pts && out, LGP_E_ARG, "null argument");
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  if (pts->n == 0) return LGP_OK;
  Plan plan = plan_for(k, pts->d);
  Module* mod = get_module(ctx, plan);
  const size_t bytes = (size_t)pts->n * 8;
  double* od = (flags & LGP_DEVICE_PTRS) ? out : (double*)ctx->scratch_get("api.diag", bytes);
  LgpGramArgs a = plan.gram;
  a.x = pts->x;
  a.y = pts->x;
  a.out = od;
  a.n_rows = pts->n;
  a.n_cols = pts->n;
  a.ld = 1;
  void* params[] = {&a};
  LGP_CU_CHECK(drv::LaunchKernel(mod->diag, (unsigned)((pts->n + 255) / 256), 1, 1, 256, 1, 1, 0,
                              (CUstream)ctx->stream, params, nullptr));
  ++ctx->launches;
  stage_out(ctx, out, od, bytes, flags);
  LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  API_END
}

int lgp_predict_quad(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* train,
                     const lgp_points* test, double noise, double rel_tol, int32_t max_iter,
                     double* quad_out, int32_t* iters_out, double* final_res_out) {
  API_BEGIN
  require(ctx && k && train && test && quad_out && iters_out && final_res_out, LGP_E_ARG,
          "null argument");
  require(train->d == test->d, LGP_E_DIM, "test inputs differ in dimension from training inputs");
  require(rel_tol > 0.0, LGP_E_ARG, "rel_tolerance must be positive");
  std::lock_guard<std::recursive_mutex> g(ctx->mu);
  ctx->activate();
  const int64_t n = train->n, T = test->n;
  if (T == 0) return LGP_OK;
  const int64_t S = (n + ctx->world - 1) / ctx->world;
  const int64_t n_alloc = S * ctx->world;
  Plan plan = plan_for(k, train->d);
  Module* mod = get_module(ctx, plan);
  const int chunk = 256;
  for (int64_t c0 = 0; c0 < T; c0 += chunk) {
    const int tc = (int)std::min<int64_t>(chunk, T - c0);
    // kstar[:, c0:c0+tc] = k(X_train, X*_chunk), n x tc (FP64, models.py:232)
    double* ks = (double*)ctx->scratch_get("pq.kstar", (size_t)n_alloc * tc * 8);
    if (n_alloc > n)
      LGP_CUDA_CHECK(cudaMemsetAsync(ks + (size_t)n * tc, 0, (size_t)(n_alloc - n) * tc * 8, ctx->stream));
    LgpGramArgs a = plan.gram;
    a.x = train->x;
    a.y = test->x + (size_t)c0 * test->d;
    a.out = ks;
    a.n_rows = n;
    a.n_cols = tc;
    a.ld = tc;
    void* params[] = {&a};
    LGP_CU_CHECK(drv::LaunchKernel(mod->gram, (unsigned)n, (unsigned)((tc + 255) / 256), 1, 256, 1, 1,
                                0, (CUstream)ctx->stream, params, nullptr));
    ++ctx->launches;
    double* xd = nullptr;
    cg_device(ctx, k, train, noise, ks, tc, rel_tol, max_iter, &xd, iters_out + c0,
              final_res_out + c0);
    double* part = (double*)ctx->scratch_get("pq.part", (size_t)vec::reduce_blocks(n, tc) * tc * 8);
    double* q = (double*)ctx->scratch_get("pq.q", (size_t)tc * 8);
    vec::quad_dot(ctx, ks, xd, n, tc, part, q);
    LGP_CUDA_CHECK(cudaMemcpyAsync(quad_out + c0, q, (size_t)tc * 8, cudaMemcpyDeviceToHost, ctx->stream));
    LGP_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  }
  API_END
}

}  // extern "C"

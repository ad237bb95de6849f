// Internal declarations shared by the C-ABI front end, the kernel-tree code
// generator / NVRTC JIT, the AOT FP64 vector kernels and the solver drivers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lightgp.h"
#include "jit/lgp_jit_abi.h"

namespace lgp {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

// driver API, resolved lazily (lgp_driver.cpp)
namespace drv {
CUresult ModuleLoadData(CUmodule* m, const void* image);
CUresult ModuleUnload(CUmodule m);
CUresult ModuleGetFunction(CUfunction* f, CUmodule m, const char* name);
CUresult FuncSetAttribute(CUfunction f, CUfunction_attribute a, int v);
CUresult FuncGetAttribute(int* v, CUfunction_attribute a, CUfunction f);
CUresult OccupancyMaxActiveBlocksPerMultiprocessor(int* n, CUfunction f, int bs, size_t smem);
CUresult LaunchKernel(CUfunction f, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                      unsigned by, unsigned bz, unsigned smem, CUstream s, void** params,
                      void** extra);
CUresult GetErrorString(CUresult r, const char** s);
}  // namespace drv

#define LGP_CUDA_CHECK(expr)                                                              \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::lgp::Error(_e == cudaErrorMemoryAllocation ? LGP_E_OOM : LGP_E_CUDA,        \
                         std::string(#expr) + ": " + cudaGetErrorString(_e));             \
  } while (0)

#define LGP_CU_CHECK(expr)                                                                \
  do {                                                                                    \
    CUresult _r = (expr);                                                                 \
    if (_r != CUDA_SUCCESS) {                                                             \
      const char* _s = nullptr;                                                           \
      ::lgp::drv::GetErrorString(_r, &_s);                                                          \
      throw ::lgp::Error(_r == CUDA_ERROR_OUT_OF_MEMORY ? LGP_E_OOM : LGP_E_CUDA,        \
                         std::string(#expr) + ": " + (_s ? _s : "?"));                   \
    }                                                                                     \
  } while (0)

// ---------------------------------------------------------- kernel trees
struct Node {
  int kind;
  double p[2];
};

struct Tree {
  std::vector<Node> nodes;  // pre-order
  bool has_linear() const;
};

int node_arity(int kind);
int node_nparams(int kind);

// Tuning of one matvec module (compile-time constants of the JIT kernel).
struct Tuning {
  int tb = 1;        // RHS per pass
  int r = 8;         // rows per thread
  int threads = 256; // CTA size
  int cc = 64;       // columns per shared-memory tile
  int stages = 4;    // TMA pipeline depth
  int minb = 1;      // __launch_bounds__ min blocks
};

// Output of the code generator for (tree structure, D, TB, flags).
struct Plan {
  std::string key;          // cache key = full source text + options
  std::string source;       // NVRTC source
  Tuning tune;
  int d = 0, fr = 0, fc = 0;
  bool signed_vals = false;
  double root_scale = 1.0;  // product of Scale nodes on the root chain (FP64 epilogue)
  LgpPrepArgs prep{};       // pc[] filled
  LgpMatvecArgs mv{};       // kc[] filled
  LgpGramArgs gram{};       // pc[] filled (includes the root scale)
  size_t smem_bytes = 0;
  // tensor-core variant (tcgen05 3xTF32): r^2-stationary trees, D >= 4, t >= 8
  bool tc = false;
  int tc_kd = 0;            // K of the distance GEMM in FP16 halves (3D + 4, multiple of 16)
  int tc_n = 16;            // RHS per pass (GEMM2 N)
  int tc_fw = 0;            // FP32 features per point for FMA-pipe distance chunks
  int tc_pf = 0;            // of which Periodic (cos, sin) features, from offset P0
  size_t smem_tcsym = 0;    // dynamic shared memory of lgp_matvec_tcsym (at R = kTsRMax)
  size_t smem_tcsym_fixed = 0;  // ... without the [2R][64] column accumulators
  int ts_rmax = 0;              // largest super-tile R that fits the shared memory
  int ts_nwg = 3;           // lgp_matvec_tcsym epilogue warpgroups
  LgpTcArgs tca{};          // kc[] filled
};

Plan make_plan(const Tree& tree, int d, int tb, uint32_t flags);
// The tensor-core plan for the same tree, or a plan with tc == false when the
// tree / shape is not eligible (see lgp_codegen.cpp).
Plan make_tc_plan(const Tree& tree, int d, int t, uint32_t flags);
// Sensitivity of the tree to its squared distances: sum over r^2 leaves of
// 1.5 / lengthscale^2 (bounds |dk/d r^2| of RBF, Matern-3/2 and -5/2 leaves).
double r2_gain(const Tree& tree);
// The norm-trick distances (|c|^2 + |c'|^2 - 2 c.c', FP32 / FP16x2) lose
// ~2^-22 (|c| + |c'|)^2 absolutely; point sets whose reach (in lengthscales)
// exceeds this bound use direct differences instead (MatvecOp::prepare).
constexpr double kNormTrickReach2 = 210.0;
// K1-TC-sym super-tiles: at most this many row blocks per work item (its
// [2R][64] FP64 column accumulators live in shared memory)
constexpr int kTsRMax = 64;

// A loaded JIT module.
struct Module {
  CUmodule mod = nullptr;
  CUfunction prep = nullptr, matvec = nullptr, gram = nullptr, diag = nullptr;
  CUfunction matvec_sym = nullptr;  // symmetric-operator K1 (SIMT modules)
  CUfunction tcsym = nullptr;       // symmetric tensor-core K1, t = 1 (TC modules)
  bool tc = false;  // module holds lgp_tc_prep / lgp_matvec_tc in prep / matvec
  int blocks_per_sm = 1;
  int regs = 0;
  std::string log;
};

// Compile (or fetch from the in-memory / on-disk cache) the module for a plan.
Module* get_module(struct Context* ctx, const Plan& plan);

// ------------------------------------------------------------- contexts
struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
};

struct Comm;  // NCCL communicator (dlopen'ed), null for world == 1

// K1-TC-sym work item: row blocks [Ia, Ib) x 64-column chunks [ca, cb) of
// the pair triangle c >= 2I, `pairs` (I, c) tiles of 128 x 64 entries
struct TsRect {
  int Ia, Ib, ca, cb;
  int64_t pairs;
};
std::vector<TsRect> ts_items(int n_rb, int n_tiles, int R, int slots);
// the items of one operator shape: R, this rank's item range, the item table
// [n_items][6] and the record lists of the epilogue (see MatvecOp::prepare)
struct TsSchedule {
  int R = 1, n_items = 0, item_lo = 0, item_hi = 0, nrr = 0, ncr = 0;
  std::vector<int> it, idx;
};

struct Context {
  int device = 0;
  int rank = 0;
  int world = 1;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  Comm* comm = nullptr;
  // row-sharded schedule (local rows + NCCL all-gather): every multi-rank
  // context, and a one-rank context opened with an NCCL id (GPU test of the
  // sharded path on one device)
  bool sharded() const { return comm != nullptr; }
  std::recursive_mutex mu;
  std::map<std::string, std::unique_ptr<Module>> modules;
  std::map<std::string, DeviceBuffer> scratch;
  std::map<std::string, std::shared_ptr<TsSchedule>> ts_cache;  // K1-TC-sym schedules
  uint64_t launches = 0;
  void* flush_buf = nullptr;
  int* done_pin = nullptr;               // pinned ring of device done-flag copies (solver loops)
  cudaStream_t copy_stream = nullptr;    // staged host->device uploads (MatvecOp::run_staged)
  cudaEvent_t copy_ev[2] = {};
  cudaEvent_t done_ev[16] = {};          // ... and their completion events
  size_t flush_bytes = 0;
  // K1 timing (lgp_ctx_set_profile): event pairs around every fused-matvec
  // launch, on the launching stream
  bool profile = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool, ev_pending;
  double prof_ms = 0.0;
  uint64_t prof_count = 0;

  // stream-ordered pool for point sets (no cudaMalloc / cudaFree + sync per call)
  std::map<size_t, std::vector<void*>> pool;
  void* pool_get(size_t bytes);
  void pool_put(void* p, size_t bytes);
  static size_t pool_round(size_t bytes);

  void* scratch_get(const std::string& name, size_t bytes);  // grow-only
  void activate();  // cudaSetDevice for the calling thread
};
const TsSchedule& ts_schedule(Context* ctx, int n_rb, int n_tiles, int rmax, bool rank_split);


struct KernelHandle {
  Context* ctx;
  Tree tree;
};

struct Points {
  Context* ctx;
  int64_t n = 0;
  int32_t d = 0;
  double* x = nullptr;        // device n x d FP64, followed by ctr (one pooled block)
  double* ctr = nullptr;      // device d FP64: column mean (centring of features)
  size_t bytes = 0;           // pooled block size
  std::vector<double> center; // host copy of ctr
  double radius = 0.0;        // max_i |x_i - center| (host, FP64)
};

// ------------------------------------------------------ communicator
Comm* comm_create(int rank, int world, const uint8_t* id128, cudaStream_t stream);
void comm_destroy(Comm* c);
void comm_unique_id(uint8_t* out128);
// in-place all-gather: buf holds world slices of `count` doubles; this
// rank's slice is at buf + rank*count.
void comm_allgather_inplace(Comm* c, double* buf, size_t count, cudaStream_t stream);
// buf[0, count) <- sum over ranks, identical bits on every rank
void comm_allreduce_sum_inplace(Comm* c, double* buf, size_t count, cudaStream_t stream);
// element-wise max over ranks of `count` HOST doubles (timing / barriers; synchronous)
void comm_allreduce_max_host(Comm* c, double* vals, int count, cudaStream_t stream);

// ------------------------------------------------------ matvec engine


// Device-resident matvec: out_rows[n_rows_local x t] for rows
// [row0, row0+n_rows_local) of `rows` against all of `cols`.
// V_dev: n_cols x t (device). out_dev: n_rows_local x t (device).
// noise_v: if non-null, rows-aligned V used for the + noise·V term.
struct MatvecOp {
  Context* ctx;
  const KernelHandle* k;
  const Points* rows;
  const Points* cols;
  int64_t row0 = 0, n_rows = 0;  // local row slice
  int t = 1;
  uint32_t flags = 0;
  // prepared state
  Plan plan;
  Module* mod = nullptr;
  bool allow_tc = false;  // may use the tensor-core K1 (matvec API, Lanczos; not CG)
  int tc_t_hint = 0;      // pick K1-TC's RHS per pass as for max(t, this)
  int tiles_per_seg_hint = 0;  // column tiles per segment (0: fill whole waves)
  bool sym = false;       // square operator on one rank: symmetric block-pair kernel
  bool tcsym = false;     // square operator, t = 1, one rank: symmetric tensor-core kernel
  // multi-rank CG: every rank evaluates its share of the symmetric pair items
  // over ALL rows (K1-TC-sym), the per-rank products are all-reduced
  bool rank_split = false;
  int item_lo = 0, item_hi = 0;  // this rank's items [lo, hi) (rank_split)
  int n_items = 0;
  int ts_R = 1;                  // tcsym: max row blocks per item (record strides)
  int* items = nullptr;          // tcsym: [n_items][4] = (Ia, Ib, ca, cb), launch order
  int* recs = nullptr;           // tcsym: epilogue record lists (see prepare)
  int *r_ptr = nullptr, *r_rec = nullptr, *c_ptr = nullptr, *c_rec = nullptr;
  int n_units = 0;
  int* units = nullptr;
  double* colpart = nullptr;
  size_t smem_sym = 0;
  float* r32 = nullptr;     // K1-TC FP32 row / column features
  float* c32 = nullptr;
  float* fr = nullptr;
  float* fc = nullptr;
  double* vpack = nullptr;
  void* vtc = nullptr;
  float* vscale = nullptr;
  int* v_inexact = nullptr;
  double* partial = nullptr;
  int n_rows_pad = 0, n_cols_pad = 0, n_rb = 0, n_seg = 0, n_pass = 0, n_tiles = 0,
      tiles_per_seg = 0;
  std::string tag;

  void prepare();  // features, scratch, schedule
  void run(const double* V_dev, double* out_dev, double noise, const double* noise_v,
           const int* done);
  // K1-TC with V in (pageable or pinned) host memory: V's upload in two parts
  // on the copy stream, each part's pack + K1 launch (its column segments)
  // queued as soon as the part has landed, so the second part's transfer
  // overlaps the first part's K1. True if it ran (else the caller stages V).
  // after_copy0 runs on the host once every part's copy is queued, while the
  // first part's K1 runs (the host-side V scan); if it throws, the streams
  // are drained and the exception propagates (no result is returned).
  bool run_staged(const double* V_host, double* V_dev, double* out_dev, double noise, bool square,
                  const std::function<void()>& after_copy0);
  int tc_split() const;
  // K1-TC-sym alone, on the already packed vpack (fused CG iteration)
  void tcsym_kernel(const int* done);
};

// ------------------------------------------------------ solver drivers
// Host view of a solver loop's device `done` flag without stalling the GPU:
// check() queues an asynchronous copy of the flag into pinned memory (+ an
// event) and returns true once an already completed copy shows the flag set;
// at most `ahead` copies stay in flight (the host then waits for the oldest),
// so the host runs a bounded number of iterations ahead and iterations
// enqueued past convergence exit at their first instruction.
struct DonePoller {
  Context* ctx;
  const int* done_dev;
  int ahead;
  int head = 0, tail = 0;  // queued copies [head, tail) in the ring
  DonePoller(Context* c, const int* d, int a);
  bool check();
  bool drain();  // wait for every queued copy; true if any shows done
};
std::pair<cudaEvent_t, cudaEvent_t> k1_event_begin(Context* ctx);
void k1_event_end(Context* ctx, std::pair<cudaEvent_t, cudaEvent_t> ev);
// shifted systems riding on a single-RHS CG (lgp_cg_shifted): solutions of
// (K + (noise + sig[e]) I) x_e = b, sig[e] >= 0 (host array), into xs_dev
// (n x n_sh, device); per-shift iterations / residuals to the host arrays
struct CgShifts {
  int n = 0;
  const double* sig = nullptr;
  double* xs_dev = nullptr;
  int32_t* iters = nullptr;
  double* res = nullptr;
};
void cg_device(Context* ctx, const KernelHandle* k, const Points* pts, double noise,
               const double* B_dev, int t, double rel_tol, int max_iter, double** x_dev,
               int32_t* iters_out, double* res_out, const CgShifts* shifts = nullptr);
void lanczos_device(Context* ctx, const KernelHandle* k, const Points* pts, double noise,
                    const double* Z_dev, int t, int steps, double* alphas, double* betas,
                    int32_t* steps_out);
std::string jit_compile(const std::string& source, std::string* log_out);

// ------------------------------------------------------ AOT FP64 kernels
// internal matvec flag (beside the public LGP_* bits): the tensor-core kernel
// for any RHS count (the lgp_matvec API)
constexpr uint32_t kTcAnyT = 1u << 30;

namespace vec {
// dst += src (elementwise, stream-ordered; no launch accounting: comm helper)
void add_inplace(double* dst, const double* src, int64_t n, cudaStream_t stream);
int reduce_blocks(int64_t n, int t);
void pack_rhs(Context* c, const double* V, int64_t n, int t, int64_t n_pad, int tb, int n_pass,
              double* out, const int* done);
// RHS tiles for the tensor-core K1: [n_pass][n_tiles][hi,lo][tbn x 64] TF32 split,
// UMMA K-major canonical layout
void pack_rhs_tc(Context* c, const double* V, int64_t n, int t, int n_tiles, int tbn, int n_pass,
                 void* out, float* scale, int* inexact, const int* done);
// symmetric tensor-core K1 (t = 1): out_i = scale * (column records of
// chunk(i): c_rec[c_ptr[c] .. c_ptr[c+1]) + row records of block(i):
// r_rec[r_ptr[I] .. r_ptr[I+1])) + noise * v_i, records in list order
// (fixed order: deterministic)
void tcsym_epilogue(Context* c, const double* rowpart, const double* colpart, const int* r_ptr,
                    const int* r_rec, const int* c_ptr, const int* c_rec, int64_t n, double scale,
                    double noise, const double* noise_v, double* out, const int* done);
void epilogue(Context* c, const double* partial, int n_seg, int n_pass, int64_t rows_pad, int tb,
              int64_t n_rows, int t, double scale, double noise, const double* noise_v,
              double* out, const int* done);
// symmetric kernel: out_i = sum_{J>=B} rowp[(B,J)] + sum_{I<B} colp[(I,B)], fixed order
void sym_epilogue(Context* c, const double* rowp, const double* colp, int nb, int rb, int n_pass,
                  int tb, int64_t n, int t, double scale, double noise, const double* noise_v,
                  double* out, const int* done);
// column dots: part[blk][t] then final[t] (deterministic order)
void dot_partial(Context* c, const double* a, const double* b, int64_t n, int t, double* part,
                 const int* done);
void dot_final(Context* c, const double* part, int nblk, int t, double* out, const int* done);
void fill(Context* c, double* p, int64_t n, double v);
// point-set statistics on the device: ctr[d] = column means (fixed-order
// reduction); stats[d + 2] = [means | max |x_i - mean|^2 | non-finite flag];
// scratch >= reduce_blocks(n, 1) * d doubles
void point_stats(Context* c, const double* x, int64_t n, int d, double* ctr, double* scratch,
                 double* stats);

// CG (solvers.py:87-123), see lgp_vec.cu
struct CgState {
  double* rs;      // [t]
  double* tol;     // [t]
  double* step;    // [t]
  double* beta;    // [t]
  double* res;     // [t]
  int* active;     // [t]
  int* iters;      // [t]
  int* status;     // [1]: 0 ok, 1 breakdown
  int* done;       // [1]
  int* bad_col;    // [1]
};
// multi-shift CG (see lgp_vec.cu): per-shift scalars, double-buffered by
// iteration parity
constexpr int kMaxShifts = 64;
struct CgShiftState {
  double z[kMaxShifts], zm1[kMaxShifts], res[kMaxShifts];
  double am1, bm1;  // the seed's alpha_{k-1}, beta_{k-1}
  int active[kMaxShifts], iters[kMaxShifts];
};
void cg_shift_init(Context* c, const double* b, int64_t n, int nsh, double* xs, double* ps,
                   CgShiftState* st);
void cg_shift(Context* c, double* xs, double* ps, const double* r, int64_t n, int nsh,
              const double* sig, CgShiftState* st, CgState s, int it);
void cg_init(Context* c, const double* b, double* x, double* r, double* p, int64_t n, int t,
             double rel_tol, const double* bb_final, CgState s);
void cg_fin_pap(Context* c, const double* part, int nblk, int t, CgState s);
// fused single-RHS CG (4 launches per iteration, see lgp_vec.cu): part holds
// the per-block shares (>= max(n_tiles, cg1_blocks(n)) doubles), counter one
// zero-initialised unsigned (each fused kernel's last block resets it)
void cg1_pack(Context* c, double* p, const double* r, double* vpack, int64_t n, int64_t n_pad,
              CgState s);
void tcsym_epilogue_cg(Context* c, const double* rowpart, const double* colpart, const int* r_ptr,
                       const int* r_rec, const int* c_ptr, const int* c_rec, int64_t n,
                       double scale, double noise, const double* p, double* out, double* part,
                       unsigned* counter, CgState s);
int cg1_blocks(int64_t n);
// the device can hold cg1_vec's whole grid at once (else the 3-kernel step)
bool cg1_vec_supported(Context* c, int64_t n);
// the whole single-RHS CG vector step in one cooperative launch (records ->
// Ap, p.Ap, step, x / r update, r.r, beta / convergence, p and the K1
// operand); bar: 2 unsigned, zeroed once
void cg1_vec(Context* c, const double* rowpart, const double* colpart, const int* r_ptr,
             const int* r_rec, const int* c_ptr, const int* c_rec, int64_t n, int64_t n_pad, double scale,
             double noise, double* x, double* r, double* p, double* ap, double* vpack, double* part_pap,
             double* part_rs, unsigned* bar, int it, int max_iter, CgState s,
             unsigned long long* trace = nullptr);
// dst[i][k] = src[i][map[k]] for k < t_run (src n x t) / dst[i][map[k]] = src[i][k]
void gather_cols(Context* c, const double* src, int64_t n, int t, const int* map, int t_run,
                 double* dst, const int* done);
void scatter_cols(Context* c, const double* src, int64_t n, int t_run, const int* map, int t,
                  double* dst, const int* done);
void cg1_pap(Context* c, const double* p, const double* ap, int64_t n, double* part,
             unsigned* counter, CgState s);
void cg1_update(Context* c, double* x, double* r, const double* p, const double* ap, int64_t n,
                double* part, unsigned* counter, int it, int max_iter, CgState s);
void cg_update_xr(Context* c, double* x, double* r, const double* p, const double* ap, int64_t n,
                  int t, CgState s, double* part);
void cg_fin_rs(Context* c, const double* part, int nblk, int t, int it, int max_iter, CgState s);
void cg_update_p(Context* c, double* p, const double* r, int64_t n, int t, CgState s);

// Lanczos (solvers.py:126-154), see lgp_vec.cu
struct LzState {
  double* alpha;   // [t][steps]
  double* beta;    // [t][steps]
  double* a_cur;   // [t]
  double* h;       // [steps][t]
  double* nrm;     // [t]
  int* active;     // [t]
  int* count;      // [t]
  int* done;       // [1]
};
void lz_init(Context* c, const double* z, double* q0, int64_t n, int t, const double* zz_final,
             LzState s);
void lz_fin_alpha(Context* c, const double* part, int nblk, int t, int j, int steps, LzState s);
void lz_update1(Context* c, double* w, const double* q, const double* qprev, int64_t n, int t,
                int j, int steps, LzState s);
void lz_multidot(Context* c, const double* basis, int64_t stride, int nb, const double* w,
                 int64_t n, int t, double* part, const int* done);
void lz_fin_h(Context* c, const double* part, int nblk, int nb, int t, LzState s);
void lz_update2(Context* c, double* w, const double* basis, int64_t stride, int nb, int64_t n,
                int t, LzState s, double* part);
void lz_fin_beta(Context* c, const double* part, int nblk, int t, int j, int steps, LzState s);
void lz_normalize(Context* c, const double* w, double* qnext, int64_t n, int t, LzState s);
void quad_dot(Context* c, const double* a, const double* b, int64_t n, int t, double* part,
              double* out);
}  // namespace vec

}  // namespace lgp

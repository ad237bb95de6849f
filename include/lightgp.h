/*
 * lightgp.h — C ABI of the B200-native matrix-free K_y·V / CG / SLQ hot path.
 *
 * This is the drop-in boundary. The reference (minigp, pure Python) has no FFI:
 * its hot path sits behind three Python contracts that this
 * library replaces one-for-one:
 *
 *   lgp_matvec   <- minigp.solvers.matrix_free_matvec     solvers.py:57-84
 *                   (+ the slab loop over Kernel._gram     kernels.py:65-378)
 *   lgp_cg       <- minigp.solvers.cg_solve, when `apply` is the kernel
 *                   operator built by gp_fit / _operator    solvers.py:87-123,
 *                                                           models.py:183,203-213
 *   lgp_lanczos  <- the per-probe loop of slq_logdet /
 *                   _lanczos_quadrature (all probes in lockstep; the
 *                   eigh_tridiagonal quadrature stays on the host)
 *                                                           solvers.py:126-179
 *   lgp_gram     <- minigp.kernels.kernel_eval              kernels.py:381-395
 *   lgp_diag     <- minigp.kernels.kernel_diag              kernels.py:398-400
 *   lgp_kernel_compile <- the Kernel node protocol
 *                   (_params pre-order, kernels.py:73-74,225-226,298-299,333-334,368-369)
 *
 * Conventions
 *  - Every entry point returns an int status (LGP_OK = 0). On failure a
 *    thread-local message is available from lgp_last_error(). Status codes map
 *    onto minigp.errors (errors.py:9-50): LGP_E_DIM -> DimensionMismatchError,
 *    LGP_E_NONFINITE -> NonFiniteError, LGP_E_NOT_SPD -> OperatorNotSpdError,
 *    LGP_E_ARG -> ValueError, everything else -> MiniGpError / RuntimeError.
 *  - Arrays are float64, C-contiguous, row-major. Multi-RHS blocks V / out are
 *    n x t row-major (the t right-hand sides of one point are contiguous).
 *  - By default pointers are HOST pointers (caller-owned; the library copies
 *    in and out). With LGP_DEVICE_PTRS in `flags` they are device pointers on
 *    the context's GPU (e.g. from lgp_device_alloc).
 *  - One context = one GPU = one rank. With world > 1 the rows of K are
 *    sharded across ranks and every rank returns the full result (NCCL
 *    all-gather of the product slices over NVLink).
 *  - Calls on one context are serialised by an internal mutex.
 */
#ifndef LIGHTGP_H_
#define LIGHTGP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LGP_ABI_VERSION 1

/* status codes */
#define LGP_OK 0
#define LGP_E_ARG 1         /* ValueError */
#define LGP_E_DIM 2         /* DimensionMismatchError */
#define LGP_E_NONFINITE 3   /* NonFiniteError */
#define LGP_E_NOT_SPD 4     /* OperatorNotSpdError */
#define LGP_E_CUDA 5
#define LGP_E_NCCL 6
#define LGP_E_OOM 7
#define LGP_E_COMPILE 8     /* NVRTC failure while compiling a kernel tree */
#define LGP_E_UNSUPPORTED 9

/* kernel-tree node kinds, pre-order (node before children, left first) */
#define LGP_NODE_RBF 0      /* params: lengthscale            kernels.py:56-83  */
#define LGP_NODE_MATERN12 1 /* params: lengthscale            kernels.py:86-114 */
#define LGP_NODE_MATERN32 2 /* params: lengthscale            kernels.py:117-151 */
#define LGP_NODE_MATERN52 3 /* params: lengthscale            kernels.py:154-189 */
#define LGP_NODE_PERIODIC 4 /* params: lengthscale, period    kernels.py:192-235 */
#define LGP_NODE_LINEAR 5   /* params: variance               kernels.py:238-273 */
#define LGP_NODE_SCALE 6    /* params: outputscale; 1 child   kernels.py:276-308 */
#define LGP_NODE_SUM 7      /* no params; 2 children          kernels.py:311-343 */
#define LGP_NODE_PRODUCT 8  /* no params; 2 children          kernels.py:346-378 */

/* flags */
#define LGP_DEVICE_PTRS 1u   /* V / out / B / X_out ... are device pointers */
#define LGP_ACC_FP32 2u      /* matvec: FP32 accumulation variant (default FP64) */
#define LGP_DIST_DIRECT 4u   /* matvec: direct differences instead of the norm trick */
#define LGP_FORCE_SIMT 8u    /* matvec: never use the tensor-core (tcgen05) kernel */
#define LGP_NO_SYM 16u       /* matvec: no symmetric block-pair kernel for the square operator */
#define LGP_INPUTS_FINITE 32u /* caller already validated host inputs as finite (skip the scan) */

typedef struct lgp_ctx lgp_ctx;
typedef struct lgp_kernel lgp_kernel;
typedef struct lgp_points lgp_points;

/* ---- library / context ------------------------------------------------ */
int lgp_abi_version(void);
const char* lgp_last_error(void);
int lgp_device_count(int* out);
/* Row partition of n rows over `world` ranks: [*r0, *r1) for `rank`; every
 * rank's slice has ceil(n/world) rows of storage (the last may be short). */
int lgp_partition(int64_t n, int world, int rank, int64_t* r0, int64_t* r1);
/* NCCL unique id (128 bytes) for a multi-rank context; call on rank 0 and
 * broadcast the bytes to the other ranks out of band. */
int lgp_comm_unique_id(uint8_t* out128);
/* world == 1: nccl_id may be NULL (no communicator). A non-NULL id at world 1
 * opens a one-rank NCCL communicator and runs the row-sharded schedule
 * (device coverage of the multi-GPU path on one GPU). TEST ONLY: an id whose
 * first 12 bytes are "LGP-LOOPBACK" makes the ranks of one process (host
 * threads, one context each, same GPU) a loopback group with host-mediated
 * gathers (tests/test_gpu_loopback.py). */
int lgp_ctx_create(int device, int rank, int world, const uint8_t* nccl_id, lgp_ctx** out);
/* Element-wise max over the context's ranks of count HOST doubles, in place
 * (NCCL all-reduce on the context's communicator; synchronous). A context
 * without a communicator leaves vals unchanged. Used for max-over-ranks
 * timings and as a barrier (count = 1). */
int lgp_comm_allreduce_max(lgp_ctx* ctx, double* vals, int32_t count);
int lgp_ctx_destroy(lgp_ctx* ctx);
int lgp_ctx_sync(lgp_ctx* ctx);
/* number of kernels this library has launched on the context (for bench) */
int lgp_ctx_launch_count(lgp_ctx* ctx, uint64_t* out);
/* Per-launch CUDA-event timing of the fused K1 matvec kernel (on its own
 * stream): total device ms and launch count since the last reset. */
int lgp_ctx_set_profile(lgp_ctx* ctx, int on);
int lgp_ctx_profile(lgp_ctx* ctx, double* k1_ms_total, uint64_t* k1_launches, int reset);
/* CUDA-event timer on the context's stream */
int lgp_timer_start(lgp_ctx* ctx);
int lgp_timer_stop(lgp_ctx* ctx, float* ms);
/* device memory owned by the caller, on the context's GPU */
int lgp_device_alloc(lgp_ctx* ctx, size_t bytes, void** out);
int lgp_device_free(lgp_ctx* ctx, void* ptr);
int lgp_memcpy_h2d(lgp_ctx* ctx, void* dst, const void* src, size_t bytes);
int lgp_memcpy_d2h(lgp_ctx* ctx, void* dst, const void* src, size_t bytes);
/* page-locked host memory (for host<->device copies at full PCIe speed) */
int lgp_host_alloc(size_t bytes, void** out);
int lgp_host_free(void* ptr);
/* *all_finite = 1 iff none of p[0..n) is NaN or +-Inf (host scan, several
   threads for large arrays; needs no GPU). The Python layer's input checks
   (linalg.as_matrix / as_vector, reference linalg.py:91-106) use it. */
int lgp_all_finite(const double* p, size_t n, int* all_finite);
/* write `bytes` to a scratch buffer (L2 flush between timed iterations) */
int lgp_flush_l2(lgp_ctx* ctx, size_t bytes);

/* ---- kernel trees ------------------------------------------------------ */
/* kinds[n_nodes] pre-order; params[n_params] in _params() pre-order order.
 * ctx may be NULL (trees are not bound to a device). */
int lgp_kernel_compile(lgp_ctx* ctx, int n_nodes, const int32_t* kinds,
                       const double* params, int n_params, lgp_kernel** out);
int lgp_kernel_free(lgp_kernel* k);
/* Generated CUDA source of the module used for inputs of dimension d with t
 * right-hand sides (diagnostics / offline nvcc). Host only. */
int lgp_kernel_source(const lgp_kernel* k, int32_t d, int32_t t, uint32_t flags, char* buf,
                      size_t cap, size_t* needed);
/* NVRTC-compile that module into the on-disk cubin cache and return the
 * ptxas log (registers / spills). Host only: needs no GPU. */
int lgp_kernel_jit(const lgp_kernel* k, int32_t d, int32_t t, uint32_t flags, char* log,
                   size_t cap);

/* ---- point sets ---------------------------------------------------------- */
/* X: n x d float64 host array; validated finite. Copied to the device. */
int lgp_points_upload(lgp_ctx* ctx, const double* X, int64_t n, int32_t d, lgp_points** out);
int lgp_points_free(lgp_points* p);

/* ---- hot path ------------------------------------------------------------ */
/* out[n_rows x t] = K(rows, cols) · V[n_cols x t]  (+ noise · V when rows == cols)
 * matrix_free_matvec semantics (solvers.py:57-84) for t right-hand sides. */
int lgp_matvec(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* rows,
               const lgp_points* cols, double noise, const double* V, int32_t t,
               double* out, uint32_t flags);

/* Multi-RHS CG on (K + noise I) with per-column semantics identical to
 * cg_solve (solvers.py:87-123): zero column -> 0 iterations; stop when
 * sqrt(r.r) <= rel_tol * ||b||; max_iter <= 0 means min(n, 1000);
 * pAp <= 0 -> LGP_E_NOT_SPD. B, X_out: n x t. iters_out, final_res_out: t. */
int lgp_cg(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* pts, double noise,
           const double* B, int32_t t, double rel_tol, int32_t max_iter, double* X_out,
           int32_t* iters_out, double* final_res_out, uint32_t flags);

/* Multi-shift CG: solves (K + (noise + shifts[e]) I) x_e = b for all e <
 * n_shifts (<= 64) with ONE matvec per iteration - the shifted systems share
 * the seed's Krylov space and residual direction (CG-M, Jegerlehner 1996);
 * each stops on its own recurrence residual (solvers.py:114-119 per solve).
 * noise: the seed system's (the smallest); shifts[e] >= 0 relative to it.
 * X_out: n x n_shifts row-major; iters_out / final_res_out: n_shifts. Used
 * by the optimiser for the 2P + 1 evaluations that differ only in the root
 * output scale and the noise. */
int lgp_cg_shifted(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* pts, double noise,
                   const double* b, int32_t n_shifts, const double* shifts, double rel_tol,
                   int32_t max_iter, double* X_out, int32_t* iters_out, double* final_res_out,
                   uint32_t flags);

/* Lanczos with one full CGS re-orthogonalisation pass per step from each
 * column of Z (n x t), all columns in lockstep (solvers.py:126-154).
 * alphas: t x steps, betas: t x (steps-1) (row-major, unused tail = 0),
 * steps_out[c] = number of alphas built for column c (betas: steps_out-1). */
int lgp_lanczos(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* pts, double noise,
                const double* Z, int32_t t, int32_t steps, double* alphas, double* betas,
                int32_t* steps_out, uint32_t flags);

/* Dense cross-covariance out[n_rows x n_cols] = k(rows_i, cols_j) in FP64
 * (kernel_eval, kernels.py:381-395; exactly symmetric when rows == cols). */
int lgp_gram(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* rows,
             const lgp_points* cols, double* out, uint32_t flags);
/* out[n] = k(x_i, x_i) in FP64 (kernel_diag, kernels.py:398-400). */
int lgp_diag(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* pts, double* out,
             uint32_t flags);

/* Posterior variance quadratic forms for gp_predict's CG branch
 * (models.py:236-246): quad[j] = kstar_j · (K_y^-1 kstar_j) with
 * kstar = k(X_train, X*) formed and solved on the device (multi-RHS CG,
 * one column per test point). iters_out / final_res_out: per test point. */
int lgp_predict_quad(lgp_ctx* ctx, const lgp_kernel* k, const lgp_points* train,
                     const lgp_points* test, double noise, double rel_tol, int32_t max_iter,
                     double* quad_out, int32_t* iters_out, double* final_res_out);

#ifdef __cplusplus
}
#endif
#endif /* LIGHTGP_H_ */

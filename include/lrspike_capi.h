/* lrspike C-ABI -- the drop-in boundary of the B200-native LR-SPIKE solver.
 *
 * Plain C types only (no torch, no CUDA types in signatures).  Implemented by
 * liblrspike_cuda.so (CUDA sm_100a kernels).  There is no CPU fallback: every
 * numerical operation below runs on the GPU; the host side only validates,
 * orchestrates launches and runs the Krylov scalar recurrences.
 *
 * Each entry point replaces one operation of the reference's C++ interface
 * (reference paths relative to /root/reference):
 *   lrs_mat_upload_csr      CsrMatrix + validate()      proj/core/include/lrspike/matrix.hpp:22-48,
 *                                                        proj/core/src/matrix.cpp:21-37
 *   lrs_spmv                spmv / spmv_accumulate      matrix.hpp:51-54, matrix.cpp:121-136
 *   lrs_mat_band_metrics    band_metrics                matrix.hpp:58-70, matrix.cpp:138-158
 *   lrs_make_layout         make_layout
 *   lrs_factorize           factorize (extract_blocks, factorize_block, randomized_spike_svd,
 *                           build_truncated_precond)    SPEC.md:476-484 (:180, :217, :286, :367)
 *   lrs_solve_block         solve_block / solve_block_adjoint
 *   lrs_apply_precond       the factorization's preconditioner: apply_precond_I for
 *                           LR-SPIKE-I, apply_precond_T for T / OTF
 *   lrs_apply_precond_T     apply_precond_T
 *   lrs_apply_block_jacobi  apply_block_jacobi
 *   lrs_solve               solve + bicgstab / cg / GMRES(m), solve_otf for LR-SPIKE-OTF
 *                           SPEC.md:520-528, :421-436, :503-511 (GMRES: SURVEY D1)
 *   lrs_krylov              bicgstab / cg / GMRES(m) on caller operators
 *   lrs_reduced_apply       matvec_lowrank / matvec_otf / apply_truncated_precond
 *   lrs_trunc_precond_create build_truncated_precond from explicit spikes
 *   lrs_dense_qr / _svd / _gemm  the dense steps of randomized_spike_svd
 *   lrs_last_error          the exception taxonomy      proj/core/include/lrspike/errors.hpp:11-94
 *
 * Memory: pointers tagged LRS_MEM_HOST are copied by the library (the caller
 * keeps ownership); LRS_MEM_DEVICE pointers are CUDA device pointers on the
 * context's device and are used in place.  Dense blocks are column-major with
 * leading dimension ld >= rows.
 *
 * Threading: one host thread per lrs_ctx at a time.  Factor
 * handles are immutable after lrs_factorize except for the
 * communication ledger they accumulate.
 */
#ifndef LRSPIKE_CAPI_H
#define LRSPIKE_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LRS_API __attribute__((visibility("default")))

typedef struct lrs_ctx lrs_ctx;
typedef struct lrs_mat lrs_mat;
typedef struct lrs_fact lrs_fact;

/* One status per lrspike::Error subclass (errors.hpp) plus runtime codes. */
typedef enum lrs_status {
  LRS_OK = 0,
  LRS_ERR_PARSE = 1,                      /* ParseError(line)                 errors.hpp:17 */
  LRS_ERR_UNSUPPORTED_FIELD = 2,          /* UnsupportedFieldError            errors.hpp:30 */
  LRS_ERR_DIMENSION = 3,                  /* DimensionError                   errors.hpp:36 */
  LRS_ERR_SINGULAR_SCALING = 4,           /* SingularScalingError(row)        errors.hpp:41 */
  LRS_ERR_LAYOUT = 5,                     /* LayoutError                      errors.hpp:53 */
  LRS_ERR_NOT_BLOCK_TRIDIAGONAL = 6,      /* NotBlockTridiagonalError(r,c)    errors.hpp:59 */
  LRS_ERR_SINGULAR_BLOCK = 7,             /* SingularBlockError(column)       errors.hpp:73 */
  LRS_ERR_PARAMETER = 8,                  /* ParameterError                   errors.hpp:83 */
  LRS_ERR_ILL_CONDITIONED_INTERFACE = 9,  /* IllConditionedInterfaceError     errors.hpp:86 */
  LRS_ERR_BREAKDOWN = 10,                 /* BiCGStab stagnation, SPEC.md:425 (partial result kept) */
  LRS_ERR_CUDA = 11,
  LRS_ERR_OOM = 12,
  LRS_ERR_NCCL = 13,
  LRS_ERR_NOT_IMPLEMENTED = 14,           /* an option outside the GPU path (e.g. FP32 factors of pivoted blocks) */
  LRS_ERR_PRECOND_FAILURE = 15            /* LR-SPIKE-I inner solve did not converge */
} lrs_status;

typedef enum lrs_scalar { LRS_F64 = 0, LRS_C128 = 1 } lrs_scalar;
typedef enum lrs_mem { LRS_MEM_HOST = 0, LRS_MEM_DEVICE = 1 } lrs_mem;
/* Table 1 of the paper / SPEC.md:470: LR-SPIKE-T, Block Jacobi, LR-SPIKE-I, LR-SPIKE-OTF. */
typedef enum lrs_variant {
  LRS_VARIANT_T = 0,
  LRS_VARIANT_BJ = 1,
  LRS_VARIANT_I = 2,  /* apply_precond_I */
  LRS_VARIANT_OTF = 3 /* solve_otf, SPEC.md:503-511 (lrs_solve runs it; no apply) */
} lrs_variant;
typedef enum lrs_method { LRS_GMRES = 0, LRS_BICGSTAB = 1, LRS_CG = 2 } lrs_method;
typedef enum lrs_side { LRS_SIDE_T = 0, LRS_SIDE_W = 1 } lrs_side;
/* How the low-rank spikes are built:
   LRS_SPIKE_SVD       randomized SVD of the spike T_i = A_i^-1 [0; B_i] (default)
   LRS_SPIKE_COUPLING  rank-r randomized SVD of B_i / C_i, spike = r padded solves against its
                       singular vectors (BASELINE.json north_star setup (1)) */
typedef enum lrs_spike_mode { LRS_SPIKE_SVD = 0, LRS_SPIKE_COUPLING = 1 } lrs_spike_mode;

/* Ledger stages. */
enum { LRS_STAGE_REDUCED_MATVEC = 0, LRS_STAGE_PRECOND_APPLY = 1, LRS_STAGE_RECOVERY = 2 };

/* SolverConfig. */
typedef struct lrs_solver_cfg {
  int32_t variant;    /* lrs_variant */
  int32_t passes;     /* randomized SVD passes, >= 2 (default 2) */
  int64_t p;          /* partitions */
  int64_t k;          /* coupling half-bandwidth; <= 0 -> band_metrics(A).k */
  int64_t n_svd;      /* retained rank r */
  int64_t oversample; /* < 0 -> ceil(n_svd / 2) */
  uint64_t seed;      /* Omega streams (seed, partition, side) */
  /* LR-SPIKE-I inner reduced solve ("inner"): <= 0 -> 1e-12 / 200 */
  double inner_tol;
  int64_t inner_max_iters;
  /* LR-SPIKE-OTF reduced solve ("otf_redsys"): <= 0 -> 1e-8 / 500;
     escalations (tolerance / 100 each): < 0 -> 4, 0 = none */
  double otf_tol;
  int64_t otf_max_iters;
  int32_t otf_escalations;
  /* Mixed precision (paper section 4.3): the preconditioner applies read the
     off-diagonal factor tiles in FP32 (the diagonal-tile inverses and every vector stay
     FP64; the spike construction uses the FP64 factors).  0 = FP64 throughout. */
  int32_t factor_fp32;
  int32_t spike_mode; /* lrs_spike_mode */
} lrs_solver_cfg;

/* IterConfig, SPEC.md:411-414 (+ method, GMRES restart). */
typedef struct lrs_iter_cfg {
  int32_t method;      /* lrs_method */
  int32_t restart;     /* GMRES(m) */
  double tol;          /* relative residual ||b-Ax||/||b|| per column */
  int64_t max_iters;
  double breakdown_eps; /* default 1e-30 */
  const void* x0;      /* optional initial guess, same memory kind / ld as b; NULL -> 0 */
} lrs_iter_cfg;

/* SolveReport, plus the CommLedger and timings. */
typedef struct lrs_report {
  int32_t converged;
  int32_t breakdown;
  double iterations;            /* max over columns; BiCGStab has half-iteration resolution */
  int64_t precond_applications; /* batched applications */
  int64_t matvecs;
  double residual_final;        /* max over columns of ||b - A x|| / ||b|| */
  int64_t comm_messages[3];     /* per stage, this solve */
  int64_t comm_scalars[3];
  double t_solve;               /* seconds, CUDA events on the context stream */
  uint64_t seed;
  double* history;              /* caller buffer (may be NULL) */
  int64_t history_cap;
  int64_t history_len;          /* entries written (<= cap); total produced in history_total */
  int64_t history_total;
  double inner_iterations;      /* LR-SPIKE-I: inner half-iterations summed over the applies */
  int64_t inner_solves;         /* LR-SPIKE-I: inner solves (one per applied column batch) */
  /* host round trips of this solve: calls into the transport (lrs_comm), stream
     synchronizations a host-callback transport forced before them (0 with the in-library
     NCCL plane), and synchronizations to read the Krylov scalars */
  int64_t comm_calls, comm_host_syncs, scalar_syncs;
} lrs_report;

/* Read-only facts about a factorization. */
typedef struct lrs_fact_info {
  int64_t n, p, k, n_svd, l;    /* l = n_svd + oversample */
  int64_t kl, ku;               /* band of the diagonal blocks */
  int64_t nb;                   /* tile size */
  int64_t wl, wu;               /* band width in tiles */
  int64_t factor_bytes;         /* device bytes of the tiled band factors */
  int64_t lu_flops;             /* algorithmic no-fill LU flops */
  int64_t apply_bytes;          /* algorithmic bytes per apply with n_rhs = 1 */
  int32_t rank_collapsed;       /* some spike lost rank */
  int32_t variant;
  double t_factorize;           /* seconds */
  double t_lu, t_spikes, t_precond; /* stage split of t_factorize */
  double max_interface_cond;
  int32_t lu_pairs;             /* steps per bulk LU update launch: 4 (INT8, K = 512), 2, or 0 */
  int32_t pivoted;              /* some block needed row interchanges: partial-pivoting LU */
  int32_t lu_int8;              /* bulk updates ran INT8-sliced on tcgen05 (LRS_LU_I8) */
  int32_t lu_sym;               /* symmetric blocks (A == A^T bitwise, no interchanges): the LU
                                   formed the lower trailing tiles only and took each U panel
                                   from its L panel, U_KJ = diag(U_KK) L_JK^T (LRS_LU_SYM=0: off) */
} lrs_fact_info;

typedef struct lrs_error_info {
  int32_t status;
  char message[512];
  int64_t line, row, col, column, interface_index;
  double cond_estimate;
} lrs_error_info;

/* ---- context ---------------------------------------------------------------------- */
/* stream: an existing cudaStream_t (e.g. torch's current stream) or NULL to create one. */
LRS_API lrs_status lrs_ctx_create(int device, void* stream, lrs_ctx** out);
LRS_API void lrs_ctx_destroy(lrs_ctx* ctx);
LRS_API void* lrs_ctx_stream(lrs_ctx* ctx);
LRS_API lrs_status lrs_last_error(lrs_ctx* ctx, lrs_error_info* info);
LRS_API const char* lrs_status_string(lrs_status s);
/* Number of kernel launches issued by this context so far (bench accounting). */
LRS_API int64_t lrs_ctx_launch_count(lrs_ctx* ctx);
LRS_API lrs_status lrs_ctx_synchronize(lrs_ctx* ctx);
/* Optional CUDA-event timing of every kernel launch, accumulated per kernel class
 * (bench / roofline accounting).  Classes, in order: lu_diag, lu_panel, lu_update,
 * band_solve, band_solve_adjoint, spmv, iface_apply, recovery, krylov_vec, setup_misc,
 * spike_band_solve (the multi-RHS solves of the randomized spike SVD). */
#define LRS_NUM_KERNEL_CLASSES 11
/* on = 0: off; 1: every class; otherwise bit k + 1 of `on` selects class k (timing only the
 * classes asked for keeps the event-record overhead off the other launches). */
LRS_API lrs_status lrs_ctx_set_profiling(lrs_ctx* ctx, int32_t on);
/* Totals since the last reset (reset = 1 clears after reading). */
LRS_API lrs_status lrs_ctx_kernel_times(lrs_ctx* ctx, double* ms, int64_t* counts, int32_t reset);

/* ---- matrix ----------------------------------------------------------------------- */
LRS_API lrs_status lrs_mat_upload_csr(lrs_ctx* ctx, int64_t n, int64_t nnz, const int64_t* row_ptr,
                                      const int64_t* col_idx, const void* values, int32_t scalar,
                                      int32_t mem, lrs_mat** out);
LRS_API void lrs_mat_destroy(lrs_mat* m);
LRS_API lrs_status lrs_mat_band_metrics(lrs_mat* m, int64_t* ku, int64_t* kl, int64_t* k,
                                        double* diag_weight, double* band_density);
/* y = A x (accumulate = 0) or y += A x (accumulate = 1); n_rhs columns. */
LRS_API lrs_status lrs_spmv(lrs_mat* m, const void* x, int64_t ldx, void* y, int64_t ldy,
                            int64_t n_rhs, int32_t accumulate, int32_t mem);

/* ---- partition -------------------------------------------------------------------- */
LRS_API lrs_status lrs_make_layout(int64_t n, int64_t p, int64_t k, int64_t* sizes_out);

/* ---- setup ------------------------------------------------------------------------ */
LRS_API lrs_status lrs_factorize(lrs_ctx* ctx, lrs_mat* a, const lrs_solver_cfg* cfg,
                                 lrs_fact** out);
LRS_API void lrs_fact_destroy(lrs_fact* f);
LRS_API lrs_status lrs_fact_get_info(lrs_fact* f, lrs_fact_info* info);
/* Partition sizes / offsets (p entries each). */
LRS_API lrs_status lrs_fact_get_layout(lrs_fact* f, int64_t* sizes, int64_t* offsets);
/* Low-rank spike of partition i, side T (i < p-1) or W (i > 0): u n_i x r (ld n_i),
 * sigma r, v r x k (ld r).  Host buffers; any may be NULL. */
LRS_API lrs_status lrs_fact_get_spike(lrs_fact* f, int64_t partition, int32_t side, double* u,
                                      double* sigma, double* v);
/* Tiled band factor of partition i as stored on the device (tests / inspection):
 * tiles[T_i][wl+wu+1][nb*nb] column-major nb x nb tiles; the diagonal tile holds
 * inv(L_ii) strictly below and inv(U_ii) on/above the diagonal. */
LRS_API lrs_status lrs_fact_get_tiles(lrs_fact* f, int64_t partition, double* host_out,
                                      int64_t capacity_doubles, int64_t* needed_doubles);
/* Ledger totals since factorization. */
LRS_API lrs_status lrs_fact_get_ledger(lrs_fact* f, int64_t messages[3], int64_t scalars[3]);

/* ---- apply ------------------------------------------------------------------------ */
LRS_API lrs_status lrs_solve_block(lrs_fact* f, int64_t partition, const void* rhs, int64_t ld_rhs,
                                   void* x, int64_t ld_x, int64_t n_rhs, int32_t adjoint,
                                   int32_t mem);
LRS_API lrs_status lrs_apply_precond(lrs_fact* f, const void* in, int64_t ld_in, void* out,
                                     int64_t ld_out, int64_t n_rhs, int32_t mem);
LRS_API lrs_status lrs_apply_block_jacobi(lrs_fact* f, const void* in, int64_t ld_in, void* out,
                                          int64_t ld_out, int64_t n_rhs, int32_t mem);
LRS_API lrs_status lrs_apply_precond_T(lrs_fact* f, const void* in, int64_t ld_in, void* out,
                                       int64_t ld_out, int64_t n_rhs, int32_t mem);

/* ---- the reduced system ---------------------------------------- */
/* ReducedVector blocks are 2 k p x n_rhs, column-major: partition i's top tip x_{i,t} in
 * rows [2ki, 2ki + k), its bottom tip x_{i,b} in rows [2ki + k, 2k(i+1)).  kind:
 * LRS_REDUCED_MATVEC_LOWRANK (matvec_lowrank), LRS_REDUCED_MATVEC_EXACT
 * (matvec_otf = matvec_exact with the exact spike tips),
 * LRS_REDUCED_TRUNC_PRECOND (apply_truncated_precond).  Single GPU. */
enum { LRS_REDUCED_MATVEC_LOWRANK = 0, LRS_REDUCED_MATVEC_EXACT = 1, LRS_REDUCED_TRUNC_PRECOND = 2 };
LRS_API lrs_status lrs_reduced_apply(lrs_fact* f, int32_t kind, const void* x, int64_t ldx,
                                     void* y, int64_t ldy, int64_t n_rhs, int32_t mem);

/* ---- small dense GPU operations (building blocks of randomized_spike_svd) -- */
/* Householder QR of the m x ncols block A (1 <= ncols <= 96 <= ..., ncols <= m): A is
 * overwritten by the explicit Q; R (ncols x ncols, ld ncols) is written if non-NULL. */
LRS_API lrs_status lrs_dense_qr(lrs_ctx* ctx, int32_t scalar, int64_t m, int64_t ncols, void* A,
                                int64_t lda, void* R, int32_t mem);
/* One-sided Jacobi SVD of the l x l matrix R (ld l, l <= 96; destroyed):
 * R = U diag(sigma) V^H, sigma descending, U and V l x l (ld l). */
LRS_API lrs_status lrs_dense_svd(lrs_ctx* ctx, int32_t scalar, int64_t l, void* R, void* U,
                                 void* V, double* sigma, int32_t mem);
/* C (m x n) = A (m x k) B (k x n) with k x n <= 96 x 64 (conjC: C = conj(A B)). */
LRS_API lrs_status lrs_dense_gemm(lrs_ctx* ctx, int32_t scalar, int64_t m, int64_t n, int64_t k,
                                  const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                                  int64_t ldc, int32_t conjC, int32_t mem);
/* build_truncated_precond from explicit LowRankSpikes of p partitions:
 *   uT_tips  (p-1) consecutive 2k x r blocks: the top then the bottom k-row tip of u of T_i,
 *            i = 0..p-2 (spike_tips)
 *   vT       (p-1) consecutive r x k blocks: v of T_i;  sT (p-1) x r: sigma of T_i
 *   uW_tips  (p-1) consecutive 2k x r blocks: the tips of u of W_i, i = 1..p-1
 *   vW, sW   likewise for W_i.
 * Returns a handle whose lrs_reduced_apply runs apply_truncated_precond and
 * matvec_lowrank on ReducedVectors; IllConditionedInterfaceError (interface
 * index, cond_1) when cond_1(K) or cond_1(H) of an interface exceeds 1e12. */
LRS_API lrs_status lrs_trunc_precond_create(lrs_ctx* ctx, int32_t scalar, int64_t p, int64_t k,
                                            int64_t r, const void* uT_tips, const void* vT,
                                            const double* sT, const void* uW_tips, const void* vW,
                                            const double* sW, int32_t mem, lrs_fact** out);

/* ---- solve ------------------------------------------------------------------------ */
LRS_API lrs_status lrs_solve(lrs_fact* f, lrs_mat* a, const void* b, int64_t ldb, void* x,
                             int64_t ldx, int64_t n_rhs, const lrs_iter_cfg* cfg,
                             lrs_report* report, int32_t mem);

/* ---- Krylov drivers on caller operators --------------------------- */
/* bicgstab / cg (and GMRES(m)) take abstract operator and preconditioner contracts: the
 * callback computes out = Op(in) for an n x n_rhs column-major block with leading
 * dimension ld (both DEVICE pointers on the context's device, in the scalar type of the
 * call) and returns 0, or nonzero to abort.  The library synchronizes its stream before
 * each call; the callback must finish its work (or order it on the context stream)
 * before returning. */
typedef struct lrs_operator {
  void* user;
  int32_t (*apply)(void* user, const void* in, void* out, int64_t ld, int64_t n_rhs);
} lrs_operator;
/* apply_M may be NULL (identity).  b, x: n x n_rhs blocks, mem HOST or DEVICE. */
LRS_API lrs_status lrs_krylov(lrs_ctx* c, int64_t n, int32_t scalar, const lrs_operator* apply_A,
                              const lrs_operator* apply_M, const void* b, int64_t ldb, void* x,
                              int64_t ldx, int64_t n_rhs, const lrs_iter_cfg* cfg,
                              lrs_report* report, int32_t mem);

/* ---- multi-GPU: one process per GPU, partitions sharded across the ranks ------------ */
/* Host callbacks for the exchanges of a sharded factorization.
 * Buffers are device pointers (doubles) on the caller's GPU.  The library synchronizes
 * its stream before every call and a callback must complete before it returns; every
 * rank makes the same sequence of calls.
 *   allgather: recv[q*count .. (q+1)*count) = send of rank q, for every rank q.
 *   sendrecv : send `scount` doubles to rank `dest` and receive `rcount` doubles from
 *              rank `source` (dest / source < 0: nothing to send / receive).
 * Return 0 on success. */
typedef struct lrs_comm {
  int32_t rank, size;
  void* user;
  int32_t (*allgather)(void* user, const double* send, double* recv, int64_t count);
  int32_t (*sendrecv)(void* user, const double* send, int64_t scount, int32_t dest, double* recv,
                      int64_t rcount, int32_t source);
  /* optional: both neighbour directions in one call (to_next -> rank+1 into its from_prev,
   * to_prev -> rank-1 into its from_next; NULL pointers where there is no neighbour) */
  int32_t (*neighbors)(void* user, const double* to_next, double* from_prev,
                       const double* to_prev, double* from_next, int64_t count);
  /* 1: the callbacks enqueue their transfers on the context's stream in stream order (the
   * in-library NCCL plane); the library then does not synchronize before calling them */
  int32_t stream_ordered;
} lrs_comm;

/* The in-library NCCL data plane (libnccl.so.2 loaded on first use): an lrs_comm whose
 * callbacks are grouped ncclSend / ncclRecv (both neighbour directions in one group) and
 * ncclAllGather on the context stream (stream_ordered = 1).  id: the 128-byte
 * ncclUniqueId from lrs_comm_nccl_unique_id on rank 0, shared by the launcher. */
LRS_API lrs_status lrs_comm_nccl_unique_id(void* id128);
LRS_API lrs_status lrs_comm_nccl_create(lrs_ctx* ctx, const void* id128, int32_t rank,
                                        int32_t size, lrs_comm** out);
LRS_API void lrs_comm_nccl_destroy(lrs_comm* comm);

/* Partitions [*p_lo, *p_hi) and rows [*row_lo, *row_hi) owned by `rank` (host only). */
LRS_API lrs_status lrs_shard_plan(int64_t n, int64_t p, int32_t size, int32_t rank, int64_t* p_lo,
                                  int64_t* p_hi, int64_t* row_lo, int64_t* row_hi);
/* Factorize this rank's shard: every rank passes the full matrix and the same config.
 * Applies and solves on the returned handle are collective; vectors are full-length,
 * each rank reads and writes its own rows [row_lo, row_hi) (other rows are scratch). */
LRS_API lrs_status lrs_factorize_dist(lrs_ctx* ctx, lrs_mat* a, const lrs_solver_cfg* cfg,
                                      const lrs_comm* comm, lrs_fact** out);

/* ---- microbenchmarks used by bench.py for the roofline denominators --------------- */
/* FP64 DMMA peak: runs a register-resident mma.sync f64 loop, returns TFLOP/s. */
LRS_API lrs_status lrs_bench_dmma_peak(lrs_ctx* ctx, double* tflops);
/* INT8 tensor-core peak: tcgen05.mma kind::i8 (M=128, N=256) from resident shared-memory
   operands on every SM, returns dense TOPS (the roofline denominator of lu_i8_gemm). */
LRS_API lrs_status lrs_bench_i8_peak(lrs_ctx* ctx, double* tops);

#ifdef __cplusplus
}
#endif

#endif /* LRSPIKE_CAPI_H */

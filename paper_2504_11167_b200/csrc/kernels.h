// Launchers for every device kernel of liblrspike_cuda.so.
#pragma once

#include "lrs_internal.h"

namespace lrs {

// ---- band factor geometry (device copy, passed by value) -----------------------------
struct BandGeom {
  const int64_t* off;    // partition row offsets [P]
  const int64_t* size;   // partition sizes [P]
  const int64_t* tbase;  // first tile index of partition p [P]
  const int* T;          // row tiles of partition p [P]
  const int64_t* fbase;  // first flag index of partition p [P]
  int P;                 // partitions on this GPU (local indices 0..P-1)
  int wl, wu, W;         // tiles below / above the diagonal, W = wl + wu + 1
  const int64_t* goff;   // global partition row offsets [Pg + 1]
  int p0, Pg;            // global index of local partition 0, global partition count
};

// ---- spmv.cu -------------------------------------------------------------------------
struct CoupleJob {
  int64_t r0, c0, b, dst0;
  const double* X;
  int64_t ldx;
  double* out;
  int64_t ldo;
  int ncols;
};
void launch_coupling(Ctx* c, const Mat* m, bool transposed, const CoupleJob* d_jobs, int njobs,
                     int64_t b, int ncols);

// ---- band_lu.cu ----------------------------------------------------------------------
// Scatter the diagonal blocks A_p of A into the zeroed tile storage (padding
// rows get a unit diagonal); record the first entry outside the
// block-tridiagonal pattern for coupling width k (row-major linear index).
void launch_extract_tiles(Ctx* c, const Mat* m, const BandGeom& g, double* tiles, int64_t k,
                          int64_t row_lo, int64_t row_hi, unsigned long long* d_bad);
// Tiled no-pivot band LU of all partitions (Tmax steps, look-ahead over two streams).
// status[2p] = min column needing a row interchange, status[2p+1] = min zero-pivot column.
void launch_band_lu(Ctx* c, const BandGeom& g, double* tiles, int Tmax, int* status);

// ---- band_solve.cu -------------------------------------------------------------------
// In-place multi-RHS banded triangular solve over all partitions.
// mode 0: L (forward), 1: U (backward), 2: U^T (forward), 3: L^T (backward).
// x is the global-row-layout block (n rows, ld), columns [0, nrhs) with nrhs <= MAX_RHS.
void launch_band_solve(Ctx* c, const BandGeom& g, const double* tiles, int mode, double* x,
                       int64_t ld, int nrhs, unsigned* flags, unsigned epoch, int* ticket,
                       int p_only, int ntiles);

// ---- dense_small.cu ------------------------------------------------------------------
struct QrJob {
  double* A;     // m x l column-major (in: matrix, out: explicit Q)
  int64_t m, ld;
  double* R;     // l x l column-major output (may be null)
};
void launch_householder_qr(Ctx* c, const QrJob* d_jobs, int njobs, int l);

struct SvdJob {
  double* R;      // l x l in; destroyed
  double* V;      // l x l out: right singular vectors of R (columns), sorted by sigma desc
  double* U;      // l x l out: left singular vectors of R (columns), sorted
  double* sigma;  // l out, descending
};
void launch_jacobi_svd(Ctx* c, const SvdJob* d_jobs, int njobs, int l);

// C[m x n] = A[m x k] * B[k x n] (column-major, small k, batched; one job per blockIdx.y)
struct GemmJob {
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  double* C; int64_t ldc;
  int64_t m;
  int n, k;
  int transA;     // 1: A is stored k x m and used transposed
};
void launch_small_gemm(Ctx* c, const GemmJob* d_jobs, int njobs, int64_t max_m, int max_n);

struct IfaceSetupJob {
  const double* uTb;  int64_t ld_uT;  // k x r tip of u_{T_i} (rows n_i-k..n_i-1)
  const double* uWt;  int64_t ld_uW;  // k x r tip of u_{W_{i+1}} (rows 0..k-1)
  const double* vtT;  const double* vtW; // k x r (= v^T), ld k
  const double* sT;   const double* sW;
  double* K; double* E; double* Hinv;  // r x r outputs
  double* cond;       // [2]: cond1(K), cond1(H)
  int* degenerate;
};
void launch_iface_setup(Ctx* c, const IfaceSetupJob* d_jobs, int njobs, int r, int64_t k);

// ---- precond.cu ----------------------------------------------------------------------
struct IfaceApplyJob {
  const double* vtT; const double* vtW;   // k x r
  const double* sT;  const double* sW;
  const double* K;   const double* E;  const double* Hinv;
  int64_t yb_row;    // off_i + n_i - k  (bottom tip of partition i)
  int64_t yt_row;    // off_{i+1}        (top tip of partition i+1)
  double* scT;       // r x nrhs: sigma_T .* (vT x_{i+1,t})   -> recovery of partition i
  double* scW;       // r x nrhs: sigma_W .* (vW x_{i,b})     -> recovery of partition i+1
  double* msg;       // 2 x r x MAX_RHS: [0] m_W (from partition i), [1] m_T (from partition i+1)
  int has_left, has_right;  // partition i / i+1 is on this GPU (else its message is received)
};
// Messages of the local sides: partial dots over 256-row slices, then a fixed-order sum.
void launch_iface_messages(Ctx* c, const IfaceApplyJob* d_jobs, int njobs, int r, int64_t k,
                           const double* y, int64_t ldy, int nrhs, double* work);
// Woodbury algebra from both messages -> scT / scW.
void launch_iface_solve(Ctx* c, const IfaceApplyJob* d_jobs, int njobs, int r, int nrhs);
size_t iface_work_doubles(int njobs, int r, int64_t k);
// dst[j] = sig[j] for j < r, zeroed where sig[j] < 1e-14 sig[0] (rank collapse);
// *flag = 1 if any spike collapsed.
struct SigmaJob { const double* sig; double* dst; };
void launch_sigma_trunc(Ctx* c, const SigmaJob* d_jobs, int njobs, int r, int* d_flag);
// x[row] = y[row] - uW[row,:] scW[part] - uT[row,:] scT[part] over the local rows
// [row_lo, row_hi); scT / scW hold one r x MAX_RHS block per GLOBAL partition.
void launch_recovery(Ctx* c, const BandGeom& g, int64_t n, int64_t row_lo, int64_t row_hi,
                     const double* y, int64_t ldy, double* x, int64_t ldx, int nrhs,
                     const double* uT, const double* uW, int r, const double* scT,
                     const double* scW);

// ---- krylov.cu -----------------------------------------------------------------------
struct ColScal { double v[MAX_RHS]; };
// Deterministic reductions: chunks of <= 2048 rows never straddle a partition; a dot
// product is summed per chunk in a fixed tree, per partition over its chunks in order,
// then over the GLOBAL partitions in order -- the same sequence of floating-point
// additions for any number of GPUs.
struct Chunks {
  const int64_t* start;  // [nchunks+1] global row boundaries of the local chunks
  const int* part_first; // [Pl+1] first chunk of each local partition
  int nchunks;
  int Pl;
};
// per-partition sums: persum[p * nvec*nrhs + q*nrhs + j] = sum over local partition p of
// X_q[:,j] . Y[:,j]   (X_q = X + q*strideX)
void launch_multidot_partition(Ctx* c, const Chunks& ch, const double* X, int64_t ldx,
                               int64_t strideX, int nvec, const double* Y, int64_t ldy, int nrhs,
                               double* partial, double* persum);
// out[o] = sum over the gathered per-partition blocks, in global partition order:
// blocks[rank][p][o] for p < counts[rank], stride pmax * nout per rank.
void launch_partition_total(Ctx* c, const double* blocks, const int* counts, int nranks,
                            int pmax, int nout, double* out);
void launch_axpby_cols(Ctx* c, int64_t n, int nrhs, int op, const ColScal& a, const ColScal& b,
                       const ColScal& act, double* X, int64_t ldx, const double* Y, int64_t ldy,
                       const double* Z, int64_t ldz, double* W, int64_t ldw);
void launch_multi_axpy_signed(Ctx* c, int64_t n, int nrhs, const double* V, int64_t ldv,
                              int64_t strideV, int nvec, const double* y_dev, double sign,
                              double* x, int64_t ldx);
void launch_multi_axpy(Ctx* c, int64_t n, int nrhs, const double* V, int64_t ldv,
                       int64_t strideV, int nvec, const double* y_dev, double* x, int64_t ldx);

// ---- bench ---------------------------------------------------------------------------
double run_dmma_peak(Ctx* c);

}  // namespace lrs

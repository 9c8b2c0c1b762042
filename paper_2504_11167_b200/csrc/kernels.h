// Launchers for every device kernel of liblrspike_cuda.so.
#pragma once

#include "lrs_internal.h"
#include "scalar.cuh"

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
  const int* t32_idx = nullptr;  // mixed precision: compact index of every tile slot in the
                                 // FP32 copy (-1: the slot lies outside its block)
  int sym = 0;           // band LU only: the blocks are symmetric, so the LU forms the lower
                         // trailing tiles (I >= J) and takes each U panel from its L panel,
                         // U_KJ = diag(U_KK) L_JK^T (band_lu.cu, lu_i8.cu)
};

// ---- spmv.cu -------------------------------------------------------------------------
template <class S>
struct CoupleJobT {
  int64_t r0, c0, b, dst0;
  const S* X;
  int64_t ldx;
  S* out;
  int64_t ldo;
  int ncols;
};
using CoupleJob = CoupleJobT<double>;
// transposed: use A^T (conjugated for complex: the adjoint couplings); accumulate: out +=
template <class S>
void launch_coupling_t(Ctx* c, const Mat* m, bool transposed, const CoupleJobT<S>* d_jobs,
                       int njobs, int64_t b, int ncols, bool accumulate = false);
void launch_spmv_z(Ctx* c, const Mat* m, const zc* x, int64_t ldx, zc* y, int64_t ldy, int nrhs,
                   int mode, const zc* b, int64_t ldb, int64_t row_lo = 0, int64_t row_hi = -1);

// ---- band_lu.cu ----------------------------------------------------------------------
// Scatter the diagonal blocks A_p of A into the zeroed tile storage (padding
// rows get a unit diagonal); record the first entry outside the
// block-tridiagonal pattern for coupling width k (row-major linear index).
void launch_extract_tiles(Ctx* c, const Mat* m, const BandGeom& g, double* tiles, int64_t k,
                          int64_t row_lo, int64_t row_hi, unsigned long long* d_bad);
// Tiled no-pivot band LU of all partitions (Tmax steps, look-ahead over two streams).
// status[2p] = min column needing a row interchange, status[2p+1] = min zero-pivot column.
// returns the steps per INT8-sliced tensor-core update (2 or 4; lu_i8.cu), 0 on DMMA
// sym: the blocks are symmetric (mat_is_symmetric): eligible for the symmetric schedule.
// Returns the steps per INT8 update (0: DMMA); *sym_used says whether that schedule ran.
int launch_band_lu(Ctx* c, const BandGeom& g, double* tiles, int Tmax, int* status,
                   bool sym = false, bool* sym_used = nullptr);
// dst[e] = (int)src[e] on the context stream (device arrays)
void launch_narrow_i64(Ctx* c, const int64_t* src, int* dst, int64_t cnt);
// A == A^T bitwise (pattern and values; real matrices), cached on the matrix
bool mat_is_symmetric(Ctx* c, Mat* m);
int launch_band_lu_z(Ctx* c, const BandGeom& g, zc* tiles, int Tmax, int* status,
                     bool sym = false, bool* sym_used = nullptr);
// the symmetric schedule is allowed on this geometry (wl == wu, LRS_LU_SYM != 0, no 2-SM update)
bool lu_sym_wanted(const BandGeom& g);
// the INT8 panel buffers fit the free device memory (+ pool cache) with 2 GB to spare
bool lu_i8_bytes_fit(size_t bytes);
// bytes of the digit slices of one 128 x 128 tile's K chunks for a D-step update
size_t lu_i8_chunk_bytes(int steps);
// integer-sliced (INT8 tensor core) two-step trailing update, lu_i8.cu: digit slices of one
// step pair's A panel (rows K+2..K+1+wl) and B panel (columns K+2..K+1+wu)
struct I8Panel {
  uint8_t* A;  // [P][wl][4 steps chunks][7 slices][128 x 32 UMMA core layout]
  uint8_t* B;  // [P][wu][4 steps chunks][7 slices][128 x 32]
  int* ea;     // [P][wl][128] row exponents
  int* eb;     // [P][wu][128] column exponents
};
// A + B + exponents of one update's panels; steps = 2 (pair, K = 256) or 4 (quad, K = 512)
size_t lu_i8_panel_bytes(const BandGeom& g, int steps);
void launch_lu_i8_slice(Ctx* c, cudaStream_t s, const BandGeom& g, const double* tiles, int K,
                        int steps, const I8Panel& pn);
// complex128 pairs: realified INT8 update (A' = [Ar Ai], B'_re = [Br; -Bi], B'_im = [Bi; Br])
void launch_lu_i8_slice_z(Ctx* c, cudaStream_t s, const BandGeom& g, const zc* tiles, int K,
                          const I8Panel& pn);
void launch_lu_i8_gemm_z(Ctx* c, cudaStream_t s, const BandGeom& g, zc* tiles, int K, int kind,
                         const I8Panel& pn);
size_t lu_i8_panel_bytes_z(const BandGeom& g);
// kind 3: look-ahead rows / columns K+steps .. K+2 steps-1; kind 4: the bulk (I, J >= K+2 steps)
void launch_lu_i8_gemm(Ctx* c, cudaStream_t s, const BandGeom& g, double* tiles, int K, int kind,
                       int steps, const I8Panel& pn);
bool lu_i8_2sm();  // LRS_I8_2SM=1: the bulk update on SM pairs (lu_i8_gemm2_kernel)
// the look-ahead driver, shared by the real and complex kernels
struct LuKernels {
  void (*diag)(Ctx*, cudaStream_t, const BandGeom&, void* tiles, int K, int* status);
  // kind 0: panel, 1: rest of the trailing update, 2: look-ahead row/column; with pairs:
  // 3: look-ahead row/column K+2 with steps K, K+1; 4: the rest with steps K, K+1
  void (*gemm)(Ctx*, cudaStream_t, const BandGeom&, void* tiles, int K, int* status, int kind);
  bool pairs = false;
  const I8Panel* i8 = nullptr;  // [2] (update parity): kinds 3 / 4 on the INT8 tensor cores
  int steps = 2;                // steps per INT8 update: 2 (pairs) or 4 (quads, K = 512)
  bool cplx = false;            // complex128 tiles: the realified INT8 kernels (pairs)
};
void run_band_lu(Ctx* c, const BandGeom& g, void* tiles, int Tmax, int* status,
                 const LuKernels& L);
bool lu_uses_pairs(const BandGeom& g, const LuKernels& L);
// the real LU runs two-step (rank-256) bulk updates when the band spans >= 2 tiles
bool lu_real_pairs(const BandGeom& g);
// partial pivoting (band_lu_piv.cu): ipiv [total_rowtiles * 128] partition-local pivot
// rows; perm [total_rowtiles * piv_perm_ints stride]: each step's composed permutation
void launch_band_lu_piv(Ctx* c, const BandGeom& g, double* tiles, int Tmax, int* status,
                        int* ipiv, int* perm);
void launch_lu_panel_piv(Ctx* c, cudaStream_t s, const BandGeom& g, double* tiles, int K,
                         int* ipiv, int* perm, int* status);
size_t piv_perm_ints(int64_t total_rowtiles);
// complex128 (zgbtrf / zgbtrs): the same over zc tiles; the transposed L solve is L^H
void launch_band_lu_piv_z(Ctx* c, const BandGeom& g, zc* tiles, int Tmax, int* status, int* ipiv,
                          int* perm);
void launch_lu_panel_piv_z(Ctx* c, cudaStream_t s, const BandGeom& g, zc* tiles, int K,
                           int* ipiv, int* perm, int* status);
void launch_piv_lsolve_z(Ctx* c, const BandGeom& g, const zc* tiles, const int* perm, int Tmax,
                         bool transposed, zc* x, int64_t ld, int nrhs, int p_only);
// forward L (transposed = false) or backward L^T solve with the interleaved interchanges
void launch_piv_lsolve(Ctx* c, const BandGeom& g, const double* tiles, const int* perm, int Tmax,
                       bool transposed, double* x, int64_t ld, int nrhs, int p_only);
void launch_extract_tiles_z(Ctx* c, const Mat* m, const BandGeom& g, zc* tiles, int64_t k,
                            int64_t row_lo, int64_t row_hi, unsigned long long* d_bad);

// ---- band_solve.cu -------------------------------------------------------------------
// In-place multi-RHS banded triangular solve over all partitions.
// mode 0: L (forward), 1: U (backward), 2: U^T (forward), 3: L^T (backward).
// x is the global-row-layout block (n rows, ld), columns [0, nrhs), nrhs <= SOLVE_MAX_RHS.
// flags: SOLVE_GROUPS x flag_stride ready flags (one set per 16-column group).
// t32: FP32 copy of the tiles (off-diagonal tiles read from it in modes 0 / 1) or null.
// mbox: [flag_stride][2 NB] zero-initialised handoff words of the one-RHS L / U sweeps
// The one-RHS L then U sweeps of the apply in one launch (band_solve_lu1_kernel): real,
// no interchanges, all local partitions; epochs epoch_l < epoch_u fresh for this apply.
void launch_band_solve_lu1(Ctx* c, const BandGeom& g, const double* tiles, double* x,
                           int64_t ld, unsigned epoch_l, unsigned epoch_u, int* ticket,
                           int ntiles, const float* t32, unsigned long long* mb);
void launch_band_solve(Ctx* c, const BandGeom& g, const double* tiles, int mode, double* x,
                       int64_t ld, int nrhs, unsigned* flags, unsigned epoch, int* ticket,
                       int p_only, int ntiles, int64_t flag_stride, const float* t32,
                       unsigned long long* mbox);
// The FP32 copy of the band factors (mixed-precision apply) holds only the tile slots inside
// their block, densely: t32[idx[s] * TILE_ELEMS + e] = (float)tiles[s * TILE_ELEMS + e] for
// the nslots slots s with idx[s] >= 0.
void launch_tiles_to_fp32(Ctx* c, const double* tiles, float* t32, const int* idx,
                          int64_t nslots);
constexpr int ZSOLVE_MAX_RHS = 16 * SOLVE_GROUPS;  // 96
// complex: modes 2 / 3 are the conjugate transposes U^H, L^H
void launch_band_solve_z(Ctx* c, const BandGeom& g, const zc* tiles, int mode, zc* x, int64_t ld,
                         int nrhs, unsigned* flags, unsigned epoch, int* ticket, int p_only,
                         int ntiles, int64_t flag_stride);

// ---- dense_small.cu (templated on the scalar S = double | zc) -------------------------
template <class S>
struct QrJobT {
  S* A;          // m x l column-major (in: matrix, out: explicit Q)
  int64_t m, ld;
  S* R;          // l x l column-major output (may be null)
};
// min_m: the smallest m of the jobs (tall jobs run as 8-CTA clusters)
template <class S>
void launch_householder_qr_t(Ctx* c, const QrJobT<S>* d_jobs, int njobs, int l, int64_t min_m);

template <class S>
struct SvdJobT {
  S* R;           // l x l in; destroyed
  S* V;           // l x l out: right singular vectors of R (columns), sorted by sigma desc
  S* U;           // l x l out: left singular vectors of R (columns), sorted
  double* sigma;  // l out, descending
};
template <class S>
void launch_jacobi_svd_t(Ctx* c, const SvdJobT<S>* d_jobs, int njobs, int l);

// C[m x n] = A[m x k] * B[k x n] (column-major, small k, batched; one job per blockIdx.y);
// conjC: store conj(C) (the complex v^T = conj(Q_z U_R))
template <class S>
struct GemmJobT {
  const S* A; int64_t lda;
  const S* B; int64_t ldb;
  S* C; int64_t ldc;
  int64_t m;
  int n, k;
  int conjC;
};
template <class S>
void launch_small_gemm_t(Ctx* c, const GemmJobT<S>* d_jobs, int njobs, int64_t max_m, int max_n);

template <class S>
struct IfaceSetupJobT {
  const S* uTb;  int64_t ld_uT;  // k x r tip of u_{T_i} (rows n_i-k..n_i-1)
  const S* uWt;  int64_t ld_uW;  // k x r tip of u_{W_{i+1}} (rows 0..k-1)
  const S* vtT;  const S* vtW;   // k x r (= v^T), ld k
  const double* sT;   const double* sW;
  S* K; S* E; S* Hinv;           // r x r outputs
  double* cond;       // [2]: cond1(K), cond1(H)
  int* degenerate;
};
template <class S>
void launch_iface_setup_t(Ctx* c, const IfaceSetupJobT<S>* d_jobs, int njobs, int r, int64_t k);

// ---- precond.cu ----------------------------------------------------------------------
template <class S>
struct IfaceApplyJobT {
  const S* vtT; const S* vtW;   // k x r
  const double* sT;  const double* sW;
  const S* K;   const S* E;  const S* Hinv;
  int64_t yb_row;    // off_i + n_i - k  (bottom tip of partition i)
  int64_t yt_row;    // off_{i+1}        (top tip of partition i+1)
  S* scT;            // r x nrhs: sigma_T .* (vT x_{i+1,t})   -> recovery of partition i
  S* scW;            // r x nrhs: sigma_W .* (vW x_{i,b})     -> recovery of partition i+1
  S* msg;            // 2 x r x MAX_RHS: [0] m_W (from partition i), [1] m_T (from partition i+1)
  int has_left, has_right;  // partition i / i+1 is on this GPU (else its message is received)
};
// Messages of the local sides: partial dots over 256-row slices, then a fixed-order sum.
template <class S>
void launch_iface_messages_t(Ctx* c, const IfaceApplyJobT<S>* d_jobs, int njobs, int r, int64_t k,
                             const S* y, int64_t ldy, int nrhs, S* work);
// Woodbury algebra from both messages -> scT / scW.
template <class S>
void launch_iface_solve_t(Ctx* c, const IfaceApplyJobT<S>* d_jobs, int njobs, int r, int nrhs);
size_t iface_work_doubles(int njobs, int r, int64_t k);  // in units of S
// dst[j] = sig[j] for j < r, zeroed where sig[j] < 1e-14 sig[0] (rank collapse);
// *flag = 1 if any spike collapsed.
struct SigmaJob { const double* sig; double* dst; };
// X[:, j] *= s[j] for the ncols columns of an m-row block (ld), one job per CTA
template <class S>
struct ScaleColsJobT { S* X; int64_t ld; const double* s; };
template <class S>
void launch_scale_cols_t(Ctx* c, const ScaleColsJobT<S>* d_jobs, int njobs, int64_t m, int ncols);
void launch_sigma_trunc(Ctx* c, const SigmaJob* d_jobs, int njobs, int r, int* d_flag);
// x[row] = y[row] - uW[row,:] scW[part] - uT[row,:] scT[part] over the local rows
// [row_lo, row_hi); scT / scW hold one r x MAX_RHS block per GLOBAL partition.
template <class S>
void launch_recovery_t(Ctx* c, const BandGeom& g, int64_t n, int64_t row_lo, int64_t row_hi,
                       const S* y, int64_t ldy, S* x, int64_t ldx, int nrhs, const S* uT,
                       const S* uW, int r, const S* scT, const S* scW);

// ---- reduced.cu (LR-SPIKE-I / OTF reduced system, compact 2k-per-partition layout) ----
template <class S>
void launch_tips_gather_t(Ctx* c, const BandGeom& g, int64_t k, const S* y, int64_t ldy,
                          const S* x, S* r, int64_t ldr, int nrhs);
template <class S>
void launch_tips_lowrank_t(Ctx* c, const BandGeom& g, int64_t n, int64_t k, const S* in, S* out,
                           int64_t ldr, int nrhs, const S* uT, const S* uW, int r, const S* scT,
                           const S* scW, int mode, double sign);
template <class S>
void launch_iface_scale_t(Ctx* c, const IfaceApplyJobT<S>* d_jobs, int njobs, int r, int nrhs);
void launch_coupling_present(Ctx* c, const Mat* m, const BandGeom& g, int64_t row_lo,
                             int64_t row_hi, int* d_flag);

// ---- krylov.cu -----------------------------------------------------------------------
template <class S> struct ColScalT { S v[MAX_RHS]; };
using ColScal = ColScalT<double>;
// Deterministic reductions: chunks of <= 2048 rows never straddle a partition; a dot
// product is summed per chunk in a fixed tree, per partition over its chunks in order,
// then over the GLOBAL partitions in order -- the same sequence of floating-point
// additions for any number of GPUs.
// Rows per deterministic reduction chunk of the Krylov dot products (partition aligned):
// one CTA of the partial-dot kernels per chunk.  512 rows -- 2 rows per thread -- keeps
// ~1.7k CTAs in flight on c3 (n = 884,736); with 2048-row chunks the 432 CTAs of a dot ran
// latency-bound at ~2.5x the HBM time.
constexpr int64_t KRYLOV_CHUNK = 512;
struct Chunks {
  const int64_t* start;  // [nchunks+1] global row boundaries of the local chunks
  const int* part_first; // [Pl+1] first chunk of each local partition
  int nchunks;
  int Pl;
};
// per-partition sums: persum[p * nvec*nrhs + q*nrhs + j] = sum over local partition p of
// conj(X_q[:,j]) . Y[:,j]   (X_q = X + q*strideX)
template <class S>
void launch_multidot_partition_t(Ctx* c, const Chunks& ch, const S* X, int64_t ldx,
                                 int64_t strideX, int nvec, const S* Y, int64_t ldy, int nrhs,
                                 S* partial, S* persum);
// out[o] = sum over the gathered per-partition blocks, in global partition order:
// blocks[rank][p][o] for p < counts[rank], stride pmax * nout per rank (doubles; a complex
// output is two independent doubles).
// y = A x on the local chunks (one CTA per chunk) plus the chunk partials of
// [X^H y, y^H y] (nvec = 2), bit-identical to spmv + launch_multidot_partition_t's partials
template <class S>
void launch_spmv_dot2_t(Ctx* c, const Mat* m, const Chunks& ch, const S* x, int64_t ldx, S* y,
                        int64_t ldy, int nrhs, const S* X, int64_t ldX, S* partial);
// persum of the chunk partials (the second half of launch_multidot_partition_t)
void launch_multidot_persum(Ctx* c, const Chunks& ch, int nout, const double* partial,
                            double* persum);
void launch_partition_total(Ctx* c, const double* blocks, const int* counts, int nranks,
                            int pmax, int nout, double* out);
template <class S>
void launch_axpby_cols_t(Ctx* c, int64_t n, int nrhs, int op, const ColScalT<S>& a,
                         const ColScalT<S>& b, const ColScal& act, S* X, int64_t ldx, const S* Y,
                         int64_t ldy, const S* Z, int64_t ldz, S* W, int64_t ldw);
// x[:, j] += sign * sum_q V_q[:, j] * y[q * nrhs + j]
template <class S>
void launch_multi_axpy_t(Ctx* c, int64_t n, int nrhs, const S* V, int64_t ldv, int64_t strideV,
                         int nvec, const S* y_dev, double sign, S* x, int64_t ldx);

// ---- csr.cu ----------------------------------------------------------------------------
// m->trow_ptr / tcol_idx / tvals from m->row_ptr / col_idx / vals (deterministic)
void launch_csr_transpose(Ctx* c, Mat* m);

// ---- bench ---------------------------------------------------------------------------
double run_dmma_peak(Ctx* c);
double run_i8_peak(Ctx* c);  // lu_i8.cu: dense INT8 tcgen05 TOPS

}  // namespace lrs

// The factorization handle (lrs_fact) and the host-side orchestration entry points.
#pragma once

#include <memory>
#include <vector>

#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

// A factorization owns a contiguous block of the P partitions: all of them on one GPU,
// or [p0, p0 + P) of Pg when sharded across GPUs (lrs_factorize_dist).  Vectors are
// full-length (global row indexing) on every GPU; each GPU reads and writes only its rows
// [row_lo, row_hi) plus the halo rows it receives from its neighbours.
struct Fact {
  Ctx* ctx = nullptr;
  Mat* mat = nullptr;
  int variant = LRS_VARIANT_T;
  int32_t scalar = LRS_F64;    // LRS_F64 | LRS_C128
  int sw = 1;                  // doubles per scalar: every S-typed buffer below is a
                               // DevBuf<double> of sw * (element count)
  int P = 1;                   // local partitions
  int Pg = 1, p0 = 0;          // global partitions, global index of local partition 0
  int64_t row_lo = 0, row_hi = 0;
  int64_t n = 0, k = 0, kl = 0, ku = 0;
  int r = 0, os = 0, l = 0, passes = 2;
  uint64_t seed = 0;
  int spike_mode = LRS_SPIKE_SVD;
  int wl = 0, wu = 0, W = 1, Tmax = 0;
  std::vector<int64_t> off, size, tbase, fbase;  // local partitions (global row offsets)
  std::vector<int64_t> goff;                     // global partition offsets [Pg + 1]
  std::vector<int> T;
  int64_t total_tiles = 0, total_rowtiles = 0;
  DevBuf<int64_t> d_off, d_size, d_tbase, d_fbase, d_goff;
  DevBuf<int> d_T;
  DevBuf<double> tiles;
  DevBuf<unsigned> flags;
  DevBuf<unsigned long long> mbox;  // one-RHS sweeps: x_t handoff words [rowtiles][2 NB]
  DevBuf<int> ticket;
  unsigned epoch = 0;
  DevBuf<int> status;
  DevBuf<unsigned long long> bad;
  // partial pivoting (band_lu_piv.cu): the blocks were factored with row interchanges
  bool pivoted = false;
  int lu_int8 = 0;  // steps per INT8-sliced LU update (2 or 4; lu_i8.cu), 0: DMMA
  bool blocks_sym = false;  // A == A^T bitwise (and LRS_LU_SYM != 0): the diagonal blocks are symmetric
  bool lu_sym = false;  // symmetric blocks: the LU formed the lower trailing tiles only
  DevBuf<int> ipiv, perm;
  // mixed precision: FP32 copy of the tiles, read for the off-diagonal tiles of the applies
  bool fp32 = false;
  DevBuf<float> tiles32;   // compact: only the tile slots inside their block (t32_idx)
  DevBuf<int> t32_idx;     // [total_tiles]: slot -> index in tiles32, or -1
  int64_t tiles32_count = 0;
  // low-rank spikes: u as n x r (global rows, ld n); v^T, sigma in GLOBAL partition slots
  DevBuf<double> uT, uW, vtT, vtW, sT, sW;
  // interfaces with at least one local side (jobs in global interface order)
  int ni = 0, iface0 = 0;      // number of jobs, global index of the first
  DevBuf<double> Kd, Ed, Hinv, cond;
  DevBuf<int> degen;
  DevBuf<double> scT, scW;     // per global partition, r x MAX_RHS
  DevBuf<unsigned char> iface_jobs;  // IfaceApplyJobT<S>[ni]
  DevBuf<unsigned char> iface_jobs_red;  // the same with compact reduced-vector tip rows
  DevBuf<double> iface_work, iface_msg;
  int job_left = -1, job_right = -1;  // jobs of the cross-GPU interfaces (or -1)
  // deterministic reductions (partition-aligned chunks, partition-ordered sums)
  std::vector<int64_t> chunk_start;
  std::vector<int> part_first;
  DevBuf<int64_t> d_chunks;
  DevBuf<int> d_part_first;
  // the compact reduced space of LR-SPIKE-I / OTF: 2k rows per partition, ld = ldr
  int64_t ldr = 0;
  std::vector<int64_t> rchunk_start;
  std::vector<int> rpart_first;
  DevBuf<int64_t> d_rchunks;
  DevBuf<int> d_rpart_first;
  // variant parameters (lrs_solver_cfg) and the LR-SPIKE-I inner-solve statistics
  double inner_tol = 1e-12, otf_tol = 1e-8;
  int64_t inner_max_iters = 200, otf_max_iters = 500;
  int otf_escalations = 4;
  bool coupled = true;  // some coupling block B_i / C_i is nonzero (OTF short-circuit)
  double inner_iterations = 0.0;
  int64_t inner_solves = 0;
  DevBuf<double> partial, persum, gather, dotout;
  std::vector<int> rank_pl;    // local partition count of every rank
  DevBuf<int> d_rank_pl;
  int pl_max = 1;
  // multi-GPU
  bool dist = false;
  lrs_comm comm{};
  // host round trips: transport calls, stream synchronizations forced by a host-callback
  // transport before them, and synchronizations to read Krylov scalars (dot products)
  int64_t comm_calls = 0, comm_syncs = 0, scalar_syncs = 0;
  DevBuf<double> xch;          // staging for neighbour exchanges
  // ledger, info
  int64_t ledger_msgs[3] = {0, 0, 0}, ledger_sc[3] = {0, 0, 0};
  lrs_fact_info info{};
  bool rank_collapsed = false;

  BandGeom geom() const {
    BandGeom g;
    g.off = d_off.get();
    g.size = d_size.get();
    g.tbase = d_tbase.get();
    g.T = d_T.get();
    g.fbase = d_fbase.get();
    g.P = P;
    g.wl = wl;
    g.wu = wu;
    g.W = W;
    g.goff = d_goff.get();
    g.p0 = p0;
    g.Pg = Pg;
    g.t32_idx = fp32 ? t32_idx.get() : nullptr;
    return g;
  }
  Chunks chunks() const {
    return Chunks{d_chunks.get(), d_part_first.get(), (int)chunk_start.size() - 1, P};
  }
  Chunks rchunks() const {
    return Chunks{d_rchunks.get(), d_rpart_first.get(), (int)rchunk_start.size() - 1, P};
  }
  unsigned next_epoch() { return ++epoch; }
  int rank() const { return dist ? comm.rank : 0; }
  int nranks() const { return dist ? comm.size : 1; }
};

// Contiguous balanced blocks of partitions per rank: [p_lo, p_hi) of rank `rank`.
void shard_plan(int64_t P, int size, int rank, int64_t* p_lo, int64_t* p_hi);

Fact* factorize(Ctx* c, Mat* m, const lrs_solver_cfg& cfg, const lrs_comm* comm);
// D-stage solve (local partitions, or local partition p_only >= 0), in place on x.
// Vectors are double* (LRS_F64) or interleaved complex128 (LRS_C128) per f->scalar.
void dstage(Fact* f, void* x, int64_t ld, int nrhs, bool adjoint, int p_only);
// M^-1 applied to in -> out on the local rows.  mode: APPLY_VARIANT (the factorization's
// own preconditioner: I, T or Block Jacobi), APPLY_BJ (D-stage only), APPLY_T.
enum { APPLY_VARIANT = 0, APPLY_BJ = 1, APPLY_T = 2 };
void apply_precond(Fact* f, const void* in, int64_t ldi, void* out, int64_t ldo, int nrhs,
                   int mode);
void solve(Fact* f, Mat* a, const void* b, int64_t ldb, void* x, int64_t ldx, int nrhs,
           const lrs_iter_cfg& cfg, lrs_report* rep);
// reduced-system operators on compact ReducedVectors (ld = f->ldr): kind 0
// matvec_lowrank, 1 matvec_otf, 2 apply_truncated_precond
void reduced_op(Fact* f, int kind, void* x, void* y, int nrhs);
// build_truncated_precond from explicit spikes (device arrays; see solver.cu)
Fact* make_trunc_precond(Ctx* c, int32_t scalar, int64_t p, int64_t k, int r, const void* uTb,
                         const void* vT, const double* sT, const void* uWt, const void* vW,
                         const double* sW);
// BiCGStab / CG / GMRES(m) on caller operators (device buffers, ld = n)
void krylov_ops(Ctx* c, int64_t n, int32_t scalar, const lrs_operator& A, const lrs_operator* M,
                const void* b, int64_t ldb, void* x, int64_t ldx, int nrhs,
                const lrs_iter_cfg& cfg, lrs_report* rep);

}  // namespace lrs

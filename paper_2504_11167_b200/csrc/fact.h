// The factorization handle (lrs_fact) and the host-side orchestration entry points.
#pragma once

#include <memory>
#include <vector>

#include "kernels.h"
#include "lrs_internal.h"

namespace lrs {

struct IfaceApplyJobDev;  // device job layout lives in precond.cu via IfaceApplyJob

struct Fact {
  Ctx* ctx = nullptr;
  Mat* mat = nullptr;
  int variant = LRS_VARIANT_T;
  int P = 1;
  int64_t n = 0, k = 0, kl = 0, ku = 0;
  int r = 0, os = 0, l = 0, passes = 2;
  uint64_t seed = 0;
  int wl = 0, wu = 0, W = 1, Tmax = 0;
  std::vector<int64_t> off, size, tbase, fbase;
  std::vector<int> T;
  int64_t total_tiles = 0, total_rowtiles = 0;
  DevBuf<int64_t> d_off, d_size, d_tbase, d_fbase;
  DevBuf<int> d_T;
  DevBuf<double> tiles;
  DevBuf<unsigned> flags;
  DevBuf<int> ticket;
  unsigned epoch = 0;
  DevBuf<int> status;
  DevBuf<unsigned long long> bad;
  // low-rank spikes (global row layout n x r, ld n) and interface data
  DevBuf<double> uT, uW, vtT, vtW, sT, sW;
  DevBuf<double> Kd, Ed, Hinv, cond;
  DevBuf<int> degen;
  DevBuf<double> scT, scW;
  DevBuf<IfaceApplyJob> iface_jobs;
  DevBuf<double> iface_work;  // partial message dots of the interface apply
  // deterministic reduction chunks (partition aligned)
  std::vector<int64_t> chunk_start;
  DevBuf<int64_t> d_chunks;
  DevBuf<double> partial, dotout;
  // apply workspace
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
    return g;
  }
  Chunks chunks() const { return Chunks{d_chunks.get(), (int)chunk_start.size() - 1}; }
  unsigned next_epoch() { return ++epoch; }
};

Fact* factorize(Ctx* c, Mat* m, const lrs_solver_cfg& cfg);
// D-stage solve (all partitions, or one partition if p_only >= 0), in place on x (ld, nrhs cols).
void dstage(Fact* f, double* x, int64_t ld, int nrhs, bool adjoint, int p_only);
// M^-1 applied to in -> out (device, ld_in / ld_out), variant T or Block Jacobi.
void apply_precond(Fact* f, const double* in, int64_t ldi, double* out, int64_t ldo, int nrhs,
                   bool block_jacobi);
void solve(Fact* f, Mat* a, const double* b, int64_t ldb, double* x, int64_t ldx, int nrhs,
           const lrs_iter_cfg& cfg, lrs_report* rep);

}  // namespace lrs

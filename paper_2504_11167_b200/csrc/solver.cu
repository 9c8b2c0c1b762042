// Host-side orchestration of the GPU path: factorize,
// apply_precond_T / apply_block_jacobi, bicgstab
// and GMRES(m).  Only launches, small
// host<->device scalar traffic and the Krylov scalar recurrences live here;
// all vector and matrix arithmetic runs in the kernels of this library.
// The control flow mirrors the CPU checker in oracle/ line by line so that the
// two produce the same iterates up to roundoff (the checker is never called).
//
// Everything is templated on the scalar S = double | zc (complex128, config c5,
// SURVEY.md D2): Hermitian dot products, complex Givens rotations, and the
// conjugate-transpose adjoint in the spike range finder.
//
// Sharding: a factorization owns partitions [p0, p0 + P) of Pg (all of them on one
// GPU).  Cross-GPU traffic is exactly the SURVEY.md 2.4 set: the two rank-r interface
// messages per apply (C1; C2 is computed on both sides, see precond.cu), the b-row
// SpMV halos (C3), the per-partition dot partials (C4, all-gathered and summed in
// global partition order, so every GPU count gives bit-identical iterates) and the
// spike tips of the cross interfaces at setup (C5).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>
#include <future>
#include <type_traits>

#include "fact.h"
#include "lrs_rng.h"

namespace lrs {

namespace {

template <class S> constexpr int SW = (int)(sizeof(S) / sizeof(double));
template <class S> S* sp(const DevBuf<double>& b) { return reinterpret_cast<S*>(b.get()); }
// host scalar of a device scalar type
template <class S>
using HT = std::conditional_t<IsC<S>::value, std::complex<double>, double>;
inline double hconj(double a) { return a; }
inline std::complex<double> hconj(std::complex<double> a) { return std::conj(a); }
inline double hreal(double a) { return a; }
inline double hreal(std::complex<double> a) { return a.real(); }
template <class S> S to_dev(HT<S> v);
template <> double to_dev<double>(double v) { return v; }
template <> zc to_dev<zc>(std::complex<double> v) { return zc{v.real(), v.imag()}; }

template <class J>
void upload(Ctx* c, DevBuf<J>& d, const std::vector<J>& h) {
  d.alloc(h.size());
  if (!h.empty()) c->stage_h2d(d.get(), h.data(), sizeof(J) * h.size());
}
template <class J>
void upload_raw(Ctx* c, DevBuf<unsigned char>& d, const std::vector<J>& h) {
  d.alloc(sizeof(J) * h.size());
  if (!h.empty()) c->stage_h2d(d.get(), h.data(), sizeof(J) * h.size());
}

template <class T>
void download(Ctx* c, T* h, const T* d, size_t count) {
  if (count == 0) return;
  LRS_CUDA(cudaMemcpyAsync(h, d, sizeof(T) * count, cudaMemcpyDeviceToHost, c->stream));
  LRS_CUDA(cudaStreamSynchronize(c->stream));
}

float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  LRS_CUDA(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

// columns [0, ncols) of a block with leading dimension ld
template <class S>
void copy_block(Ctx* c, S* dst, int64_t ldd, const S* src, int64_t lds, int64_t rows, int ncols) {
  if (rows <= 0 || ncols == 0) return;
  LRS_CUDA(cudaMemcpy2DAsync(dst, sizeof(S) * ldd, src, sizeof(S) * lds, sizeof(S) * rows, ncols,
                             cudaMemcpyDeviceToDevice, c->stream));
}

// ---- communication (no-ops on a single GPU) ---------------------------------------------
void comm_rc(int32_t rc, const char* what) {
  if (rc != 0) throw LrsError(LRS_ERR_NCCL, std::string("communication callback failed: ") + what);
}

// Neighbour exchange of `count` doubles: to_next -> rank+1 (received there in from_prev)
// and to_prev -> rank-1 (received in from_next).  A stream-ordered transport (the
// in-library NCCL plane) enqueues both directions as one group on the context stream, so
// no host synchronization happens here; a host-callback transport gets a drained stream.
void neighbor_exchange(Fact* f, const void* to_next, void* from_prev, const void* to_prev,
                       void* from_next, int64_t count) {
  if (!f->dist || count == 0) return;
  if (!f->comm.stream_ordered) {
    LRS_CUDA(cudaStreamSynchronize(f->ctx->stream));
    ++f->comm_syncs;
  }
  const int r = f->comm.rank, G = f->comm.size;
  const int next = r + 1 < G ? r + 1 : -1, prev = r > 0 ? r - 1 : -1;
  if (f->comm.neighbors) {
    ++f->comm_calls;
    comm_rc(f->comm.neighbors(f->comm.user, next >= 0 ? static_cast<const double*>(to_next) : nullptr,
                              prev >= 0 ? static_cast<double*>(from_prev) : nullptr,
                              prev >= 0 ? static_cast<const double*>(to_prev) : nullptr,
                              next >= 0 ? static_cast<double*>(from_next) : nullptr, count),
            "neighbors");
    return;
  }
  f->comm_calls += 2;
  comm_rc(f->comm.sendrecv(f->comm.user, static_cast<const double*>(to_next),
                           next >= 0 ? count : 0, next, static_cast<double*>(from_prev),
                           prev >= 0 ? count : 0, prev),
          "sendrecv");
  comm_rc(f->comm.sendrecv(f->comm.user, static_cast<const double*>(to_prev),
                           prev >= 0 ? count : 0, prev, static_cast<double*>(from_next),
                           next >= 0 ? count : 0, next),
          "sendrecv");
}

// All-gather of a small host vector (every rank contributes v.size() doubles): setup
// decisions every rank must take identically.
std::vector<double> allgather_host(Fact* f, const std::vector<double>& v) {
  if (!f->dist) return v;
  const int G = f->comm.size;
  Ctx* c = f->ctx;
  DevBuf<double> d;
  d.alloc(v.size() * (G + 1));
  std::vector<double> out(v.size() * G);
  LRS_CUDA(cudaMemcpyAsync(d.get(), v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice,
                           c->stream));
  if (!f->comm.stream_ordered) {
    LRS_CUDA(cudaStreamSynchronize(c->stream));
    ++f->comm_syncs;
  }
  ++f->comm_calls;
  comm_rc(f->comm.allgather(f->comm.user, d.get(), d.get() + v.size(), (int64_t)v.size()),
          "allgather");
  LRS_CUDA(cudaMemcpyAsync(out.data(), d.get() + v.size(), sizeof(double) * out.size(),
                           cudaMemcpyDeviceToHost, c->stream));
  LRS_CUDA(cudaStreamSynchronize(c->stream));
  return out;
}

// SpMV halo (C3): rows [row_lo - hb, row_lo) and [row_hi, row_hi + hb) of the
// full-length block x from the neighbours, hb = the band half-width of A.
template <class S>
void halo_exchange(Fact* f, S* x, int64_t ld, int nrhs) {
  if (!f->dist) return;
  const int64_t hb = std::min<int64_t>(f->mat->k, f->row_hi - f->row_lo);
  if (hb == 0 || nrhs == 0) return;
  Ctx* c = f->ctx;
  const int64_t cnt = hb * nrhs;
  S* s_next = sp<S>(f->xch);
  S* s_prev = s_next + cnt;
  S* r_prev = s_prev + cnt;
  S* r_next = r_prev + cnt;
  copy_block(c, s_next, hb, x + f->row_hi - hb, ld, hb, nrhs);
  copy_block(c, s_prev, hb, x + f->row_lo, ld, hb, nrhs);
  neighbor_exchange(f, s_next, r_prev, s_prev, r_next, cnt * SW<S>);
  const int rk = f->comm.rank;
  if (rk > 0) copy_block(c, x + f->row_lo - hb, ld, r_prev, hb, hb, nrhs);
  if (rk + 1 < f->comm.size) copy_block(c, x + f->row_hi, ld, r_next, hb, hb, nrhs);
}

// LRS_SPMV_DOT=0: BiCGStab's t = A shat and its omega dots as separate kernels
bool spmv_dot_unfused() {
  static const bool off = std::getenv("LRS_SPMV_DOT") && std::getenv("LRS_SPMV_DOT")[0] == '0';
  return off;
}

template <class S>
void spmv_s(Ctx* c, const Mat* m, const S* x, int64_t ldx, S* y, int64_t ldy, int nrhs, int mode,
            const S* b, int64_t ldb, int64_t lo, int64_t hi) {
  if constexpr (IsC<S>::value) launch_spmv_z(c, m, x, ldx, y, ldy, nrhs, mode, b, ldb, lo, hi);
  else launch_spmv(c, m, x, ldx, y, ldy, nrhs, mode, b, ldb, lo, hi);
}

// ------------------------------------------------------------------------------------
// D-stage: banded L then U solves (or U^H then L^H for the adjoint), batches of up to
// SOLVE_MAX_RHS (real) / ZSOLVE_MAX_RHS (complex) columns, all local partitions at once.
// ------------------------------------------------------------------------------------
template <class S>
void dstage_t(Fact* f, S* x, int64_t ld, int nrhs, bool adjoint, int p_only) {
  const BandGeom g = f->geom();
  const int ntiles = p_only >= 0 ? f->T[p_only] : (int)f->total_rowtiles;
  constexpr int MAXR = IsC<S>::value ? ZSOLVE_MAX_RHS : SOLVE_MAX_RHS;
  if constexpr (!IsC<S>::value) {
    // the apply's one-RHS L + U sweeps as one launch (LRS_SOLVE_FUSED=0: two launches)
    static const bool fused = !(std::getenv("LRS_SOLVE_FUSED") &&
                                std::getenv("LRS_SOLVE_FUSED")[0] == '0');
    if (fused && nrhs == 1 && !adjoint && !f->pivoted && p_only < 0 && f->ctx->solve_fma1) {
      const unsigned el = f->next_epoch(), eu = f->next_epoch();
      launch_band_solve_lu1(f->ctx, g, f->tiles.get(), x, ld, el, eu, f->ticket.get(), ntiles,
                            (f->fp32 && !f->ctx->in_setup) ? f->tiles32.get() : nullptr,
                            f->mbox.get());
      return;
    }
  }
  for (int c0 = 0; c0 < nrhs; c0 += MAXR) {
    const int nr = std::min(MAXR, nrhs - c0);
    S* xc = x + (int64_t)c0 * ld;
    for (int half = 0; half < 2; ++half) {
      const int mode = adjoint ? 2 + half : half;
      // with row interchanges the L sweeps interleave the permutations (?gbtrs)
      if (f->pivoted && (mode == 0 || mode == 3)) {
        if constexpr (IsC<S>::value)
          launch_piv_lsolve_z(f->ctx, g, sp<zc>(f->tiles), f->perm.get(), f->Tmax, mode == 3, xc,
                              ld, nr, p_only);
        else
          launch_piv_lsolve(f->ctx, g, f->tiles.get(), f->perm.get(), f->Tmax, mode == 3, xc, ld,
                            nr, p_only);
        continue;
      }
      if constexpr (IsC<S>::value)
        launch_band_solve_z(f->ctx, g, sp<zc>(f->tiles), mode, xc, ld, nr, f->flags.get(),
                            f->next_epoch(), f->ticket.get(), p_only, ntiles, f->total_rowtiles);
      else
        launch_band_solve(f->ctx, g, f->tiles.get(), mode, xc, ld, nr, f->flags.get(),
                          f->next_epoch(), f->ticket.get(), p_only, ntiles, f->total_rowtiles,
                          (f->fp32 && !f->ctx->in_setup) ? f->tiles32.get() : nullptr,
                          f->mbox.get());
    }
  }
}

// C1 across the GPU boundaries: m_W (computed left) goes right, m_T goes left; the
// messages of nr columns are the first r * nr scalars of their r x MAX_RHS slots
template <class S>
void exchange_msgs(Fact* f, int nr) {
  if (!f->dist) return;
  const int64_t blk = (int64_t)f->r * MAX_RHS;
  S* mbase = sp<S>(f->iface_msg);
  const S* to_next = f->job_right >= 0 ? mbase + (2 * f->job_right + 0) * blk : mbase;
  S* from_prev = f->job_left >= 0 ? mbase + (2 * f->job_left + 0) * blk : mbase;
  const S* to_prev = f->job_left >= 0 ? mbase + (2 * f->job_left + 1) * blk : mbase;
  S* from_next = f->job_right >= 0 ? mbase + (2 * f->job_right + 1) * blk : mbase;
  neighbor_exchange(f, to_next, from_prev, to_prev, from_next, (int64_t)f->r * nr * SW<S>);
}

// `per_iface` messages of `scalars` each for every interface this GPU owns (the GPU of
// its left partition), so the sum over the GPUs is the single-GPU count
void ledger_add(Fact* f, int stage, int64_t per_iface, int64_t scalars) {
  int64_t owned = 0;
  for (int i = f->p0; i < f->p0 + f->P; ++i)
    if (i < f->Pg - 1) ++owned;
  f->ledger_msgs[stage] += per_iface * owned;
  f->ledger_sc[stage] += per_iface * owned * scalars;
}

template <class S>
void apply_precond_t(Fact* f, const S* in, int64_t ldi, S* out, int64_t ldo, int nrhs,
                     bool block_jacobi) {
  Ctx* c = f->ctx;
  const int64_t nl = f->row_hi - f->row_lo;
  if (out != in) copy_block(c, out + f->row_lo, ldo, in + f->row_lo, ldi, nl, nrhs);
  dstage_t(f, out, ldo, nrhs, false, -1);
  const bool lowrank = !block_jacobi && f->r > 0 && f->Pg > 1;
  if (!lowrank) return;
  const int r = f->r;
  const auto* jobs = reinterpret_cast<const IfaceApplyJobT<S>*>(f->iface_jobs.get());
  for (int c0 = 0; c0 < nrhs; c0 += MAX_RHS) {
    const int nr = std::min(MAX_RHS, nrhs - c0);
    S* xc = out + (int64_t)c0 * ldo;
    launch_iface_messages_t<S>(c, jobs, f->ni, r, f->k, xc, ldo, nr, sp<S>(f->iface_work));
    exchange_msgs<S>(f, nr);
    launch_iface_solve_t<S>(c, jobs, f->ni, r, nr);
    launch_recovery_t<S>(c, f->geom(), f->n, f->row_lo, f->row_hi, xc, ldo, xc, ldo, nr,
                         sp<S>(f->uT), sp<S>(f->uW), r, sp<S>(f->scT), sp<S>(f->scW));
  }
  // CommLedger: 2 compressed messages per local-side interface in the
  // reduced solve and 2 in the recovery, r n_rhs scalars each -- 4 (p-1) r n_rhs per
  // application summed over the GPUs (every interface is counted by the GPU of its
  // left partition).
  ledger_add(f, LRS_STAGE_PRECOND_APPLY, 2, (int64_t)r * nrhs);
  ledger_add(f, LRS_STAGE_RECOVERY, 2, (int64_t)r * nrhs);
}

// ------------------------------------------------------------------------------------
// Randomized spike SVDs and the truncated preconditioner for rank r.
// Returns false (without throwing) if an interface is ill-conditioned on ANY rank,
// filling *bad_iface / *bad_cond, so the caller can apply the r-halving retry.
// ------------------------------------------------------------------------------------
// Gaussian test blocks of the spikes of partitions [plo, phi): slot 2*i + side, k x l each
// (real for both fields, as the shared generator draws them).
// Drawn on the host with the shared counter-based generator (bit-identical to the
// checker's Omega), split over host threads: every draw is a pure function of (seed,
// stream, index), so the result does not depend on the thread count.
void fill_omega(double* h, uint64_t seed, int Pg, int plo, int phi, int64_t k, int l) {
  std::memset(h, 0, sizeof(double) * (size_t)Pg * 2 * k * l);
  std::vector<std::pair<int, int>> slots;
  for (int i = plo; i < phi; ++i)
    for (int side = 0; side < 2; ++side)
      if (!((side == LRS_SIDE_T && i == Pg - 1) || (side == LRS_SIDE_W && i == 0)))
        slots.push_back({i, side});
  const int64_t per = k * l, total = per * (int64_t)slots.size();
  if (total == 0) return;
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  nt = (unsigned)std::min<int64_t>(nt, std::max<int64_t>(1, total / 65536));
  auto work = [&](int64_t e0, int64_t e1) {
    for (int64_t e = e0; e < e1; ++e) {
      const auto [i, side] = slots[e / per];
      const uint64_t key = lrs_rng_key(seed, LRS_STREAM_OMEGA + 2ull * i + side);
      h[(size_t)(2 * i + side) * per + e % per] = lrs_rng_normal(key, (uint64_t)(e % per));
    }
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, total * t / nt, total * (t + 1) / nt);
  work(0, total / nt);
  for (auto& t : th) t.join();
}
std::vector<double> make_omega(uint64_t seed, int Pg, int plo, int phi, int64_t k, int l) {
  std::vector<double> h((size_t)Pg * 2 * k * l);
  fill_omega(h.data(), seed, Pg, plo, phi, k, l);
  return h;
}

// Omega drawn into the context's page-locked staging buffer and uploaded on the copy stream
// by a host thread, both while the band LU runs: dev (real, Pg * 2 * k * l doubles) is valid
// for the main stream once it has waited for c->ev_omega.  ev_alloc orders the copy after
// whatever used dev's pool block before.  Returns false (and leaves dev alone) on any error:
// the caller then draws and copies Omega synchronously.
bool omega_upload_task(Ctx* c, double* dev, cudaEvent_t ev_alloc, uint64_t seed, int Pg, int plo,
                       int phi, int64_t k, int l) {
  const size_t cnt = (size_t)Pg * 2 * k * l;
  if (cudaSetDevice(c->device) != cudaSuccess) return false;
  if (c->omega_host_cap < cnt) {
    if (c->omega_host) cudaFreeHost(c->omega_host);
    c->omega_host = nullptr;
    c->omega_host_cap = 0;
    if (cudaMallocHost(reinterpret_cast<void**>(&c->omega_host), sizeof(double) * cnt) !=
        cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    c->omega_host_cap = cnt;
  }
  fill_omega(c->omega_host, seed, Pg, plo, phi, k, l);
  if (cudaStreamWaitEvent(c->stream_copy, ev_alloc, 0) != cudaSuccess) return false;
  if (cudaMemcpyAsync(dev, c->omega_host, sizeof(double) * cnt, cudaMemcpyHostToDevice,
                      c->stream_copy) != cudaSuccess)
    return false;
  return cudaEventRecord(c->ev_omega, c->stream_copy) == cudaSuccess;
}

template <class S>
__global__ void omega_expand_kernel(const double* __restrict__ src, S* __restrict__ dst,
                                    int64_t cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = s_real<S>(src[e]);
}

// spike_mode = coupling (BASELINE.json north_star setup (1)):
// rank-r randomized SVD of each coupling block, then the spike by r padded solves against
// its singular vectors.  Mirrors the checker's coupling_spike_svd step by step:
//   Q_B = orth(B Om_r) [+ power passes]; B^H Q_B = Q_z R_1, R_1 = U_1 S_1 V_1^H
//   => B_r = (Q_B V_1) S_1 (Q_z U_1)^H = U_B S_B V_B^H;
//   Y = A_i^-1 pad(U_B S_B) = Q_2 R_2, R_2 = U_2 S_2 V_2^H
//   => T~ = (Q_2 U_2) S_2 (V_B V_2)^H:  u = Q_2 U_2, sigma = S_2, v^T = conj(V_B V_2).
// The k x l slots of Om / Zt hold k x r blocks (ld k); Rz / Ur / Vr slots r x r (ld r);
// Y holds side T in columns [0, r) and side W in [r, 2r) (ld n).
template <class S>
void coupling_spikes(Fact* f, int r, int l, const std::vector<std::pair<int, int>>& spk,
                     const S* Om, S* Y, S* Rz, S* Ur, S* Vr, double* sig) {
  Ctx* c = f->ctx;
  Mat* m = f->mat;
  const int Pg = f->Pg;
  const int64_t n = f->n, k = f->k;
  constexpr int w = SW<S>;
  auto slot = [&](int i, int side) { return (size_t)(2 * i + side); };
  auto goff = [&](int i) { return f->goff[i]; };
  auto gsize = [&](int i) { return f->goff[i + 1] - f->goff[i]; };
  DevBuf<double> QBb, UBb, VBb, sig1b;
  QBb.alloc((size_t)Pg * 2 * k * r * w);
  UBb.alloc((size_t)Pg * 2 * k * r * w);
  VBb.alloc((size_t)Pg * 2 * k * r * w);
  sig1b.alloc((size_t)Pg * 2 * r);
  S* QB = sp<S>(QBb);
  S* UB = sp<S>(UBb);
  S* VB = sp<S>(VBb);
  const size_t kr = (size_t)k * r, ll = (size_t)l * l;
  // X (k x r, slot stride k*l or k*r) -> B X / B^H X (k x r, slot stride k*r)
  DevBuf<CoupleJobT<S>> cj;
  auto couple = [&](bool adj, const S* src, size_t src_stride, S* dst, size_t dst_stride) {
    std::vector<CoupleJobT<S>> jobs;
    for (auto [i, side] : spk) {
      CoupleJobT<S> j{};
      const bool T = side == LRS_SIDE_T;
      if (!adj) {  // B_i = A[off_i+n_i-k.., off_{i+1}..];  C_i = A[off_i.., off_i-k..]
        j.r0 = T ? goff(i) + gsize(i) - k : goff(i);
        j.c0 = T ? goff(i + 1) : goff(i) - k;
      } else {  // B_i^H, C_i^H from the CSR of A^H
        j.r0 = T ? goff(i + 1) : goff(i) - k;
        j.c0 = T ? goff(i) + gsize(i) - k : goff(i);
      }
      j.b = k;
      j.dst0 = 0;
      j.X = src + slot(i, side) * src_stride;
      j.ldx = k;
      j.out = dst + slot(i, side) * dst_stride;
      j.ldo = k;
      j.ncols = r;
      jobs.push_back(j);
    }
    upload(c, cj, jobs);
    launch_coupling_t<S>(c, m, adj, cj.get(), (int)jobs.size(), k, r);
  };
  DevBuf<QrJobT<S>> qj;
  auto orth_k = [&](S* base, size_t stride, bool keepR) {
    std::vector<QrJobT<S>> jobs;
    for (auto [i, side] : spk)
      jobs.push_back(QrJobT<S>{base + slot(i, side) * stride, k, k,
                               keepR ? Rz + slot(i, side) * ll : nullptr});
    upload(c, qj, jobs);
    launch_householder_qr_t<S>(c, qj.get(), (int)jobs.size(), r, k);
  };
  DevBuf<SvdJobT<S>> sj;
  auto svd_r = [&](double* sg) {
    std::vector<SvdJobT<S>> jobs;
    for (auto [i, side] : spk) {
      const size_t s = slot(i, side);
      jobs.push_back(SvdJobT<S>{Rz + s * ll, Vr + s * ll, Ur + s * ll, sg + s * r});
    }
    upload(c, sj, jobs);
    launch_jacobi_svd_t<S>(c, sj.get(), (int)jobs.size(), r);
  };
  DevBuf<GemmJobT<S>> gj;
  auto gemm = [&](const std::vector<GemmJobT<S>>& jobs, int64_t maxm) {
    upload(c, gj, jobs);
    launch_small_gemm_t<S>(c, gj.get(), (int)jobs.size(), maxm, r);
  };
  // (1) range of B: Q_B = orth(B Om_r) (+ (passes - 2) / 2 power passes)
  couple(false, Om, (size_t)k * l, QB, kr);
  orth_k(QB, kr, false);
  for (int pi = 0; pi < (f->passes - 2) / 2; ++pi) {
    couple(true, QB, kr, UB, kr);
    orth_k(UB, kr, false);
    couple(false, UB, kr, QB, kr);
    orth_k(QB, kr, false);
  }
  // (2) B^H Q_B = Q_z R_1 (Q_z in VB), R_1 = U_1 S_1 V_1^H
  couple(true, QB, kr, VB, kr);
  orth_k(VB, kr, true);
  svd_r(sig1b.get());
  // (3) U_B S_B = Q_B (V_1 S_1) into the padded RHS rows of Y; V_B = Q_z U_1 (into UB)
  {
    std::vector<ScaleColsJobT<S>> sc;
    for (auto [i, side] : spk) {
      const size_t s = slot(i, side);
      sc.push_back(ScaleColsJobT<S>{Vr + s * ll, r, sig1b.get() + s * r});
    }
    DevBuf<ScaleColsJobT<S>> dsc;
    upload(c, dsc, sc);
    launch_scale_cols_t<S>(c, dsc.get(), (int)sc.size(), r, r);
  }
  LRS_CUDA(cudaMemsetAsync(Y, 0, sizeof(S) * n * 2 * r, c->stream));
  {
    std::vector<GemmJobT<S>> g1, g2;
    for (auto [i, side] : spk) {
      const size_t s = slot(i, side);
      const int64_t row0 = side == LRS_SIDE_T ? goff(i) + gsize(i) - k : goff(i);
      g1.push_back(GemmJobT<S>{QB + s * kr, k, Vr + s * ll, r, Y + row0 + (int64_t)side * r * n,
                               n, k, r, r, 0});
      g2.push_back(GemmJobT<S>{VB + s * kr, k, Ur + s * ll, r, UB + s * kr, k, k, r, r, 0});
    }
    gemm(g1, k);
    gemm(g2, k);
  }
  // (4) Y = A_i^-1 pad(U_B S_B) (2r columns: the T and W sides), Y = Q_2 R_2
  dstage_t(f, Y, n, 2 * r, false, -1);
  {
    std::vector<QrJobT<S>> jobs;
    int64_t mm = n;
    for (auto [i, side] : spk) {
      jobs.push_back(QrJobT<S>{Y + goff(i) + (int64_t)side * r * n, gsize(i), n,
                               Rz + slot(i, side) * ll});
      mm = std::min(mm, gsize(i));
    }
    upload(c, qj, jobs);
    launch_householder_qr_t<S>(c, qj.get(), (int)jobs.size(), r, mm);
  }
  // (5) R_2 = U_2 S_2 V_2^H:  u = Q_2 U_2, v^T = conj(V_B V_2), sigma = S_2 (rank collapse)
  svd_r(sig);
  std::vector<GemmJobT<S>> gu, gv;
  std::vector<SigmaJob> sjobs;
  int64_t maxm = 0;
  for (auto [i, side] : spk) {
    const size_t s = slot(i, side);
    S* ubuf = side == LRS_SIDE_T ? sp<S>(f->uT) : sp<S>(f->uW);
    S* vbuf = side == LRS_SIDE_T ? sp<S>(f->vtT) : sp<S>(f->vtW);
    double* sbuf = side == LRS_SIDE_T ? f->sT.get() : f->sW.get();
    gu.push_back(GemmJobT<S>{Y + goff(i) + (int64_t)side * r * n, n, Ur + s * ll, r,
                             ubuf + goff(i), n, gsize(i), r, r, 0});
    gv.push_back(GemmJobT<S>{UB + s * kr, k, Vr + s * ll, r, vbuf + (size_t)i * k * r, k, k, r,
                             r, IsC<S>::value ? 1 : 0});
    sjobs.push_back(SigmaJob{sig + s * r, sbuf + (size_t)i * r});
    maxm = std::max(maxm, gsize(i));
  }
  gemm(gu, maxm);
  gemm(gv, k);
  DevBuf<SigmaJob> dsj;
  upload(c, dsj, sjobs);
  DevBuf<int> flag;
  flag.alloc(1);
  LRS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), c->stream));
  launch_sigma_trunc(c, dsj.get(), (int)sjobs.size(), r, flag.get());
  int hflag = 0;
  download(c, &hflag, flag.get(), 1);
  f->rank_collapsed = hflag != 0;
}

// Per-interface Woodbury factors (K, E, H^-1, cond_1; Appendix A.1 of
// SURVEY.md) and the apply-time job tables, from the spikes in f->uT/uW/vtT/vtW/sT/sW.
// Returns false (without throwing) if an interface is ill-conditioned on ANY rank.
template <class S>
bool finish_interfaces(Fact* f, int r, int* bad_iface, double* bad_cond) {
  Ctx* c = f->ctx;
  const int Pg = f->Pg, p0 = f->p0, P = f->P;
  const int64_t n = f->n, k = f->k;
  constexpr int w = SW<S>;
  auto goff = [&](int i) { return f->goff[i]; };
  auto gsize = [&](int i) { return f->goff[i + 1] - f->goff[i]; };
  (void)n;
  // interfaces with at least one local side: global i in [iface0, iface0 + ni)
  f->iface0 = std::max(0, p0 - 1);
  const int ilast = std::min(Pg - 2, p0 + P - 1);
  const int ni = std::max(0, ilast - f->iface0 + 1);
  f->ni = ni;
  const size_t rr = (size_t)r * r;
  f->Kd.alloc((size_t)std::max(ni, 1) * rr * w);
  f->Ed.alloc((size_t)std::max(ni, 1) * rr * w);
  f->Hinv.alloc((size_t)std::max(ni, 1) * rr * w);
  f->cond.alloc((size_t)std::max(ni, 1) * 2);
  f->degen.alloc((size_t)std::max(ni, 1));
  double mx = 1.0;
  int bad_i = -1;
  double bad_c = 0.0;
  if (ni > 0) {
    std::vector<IfaceSetupJobT<S>> jobs;
    for (int q = 0; q < ni; ++q) {
      const int i = f->iface0 + q;
      IfaceSetupJobT<S> j{};
      j.uTb = sp<S>(f->uT) + goff(i) + gsize(i) - k;
      j.ld_uT = n;
      j.uWt = sp<S>(f->uW) + goff(i + 1);
      j.ld_uW = n;
      j.vtT = sp<S>(f->vtT) + (size_t)i * k * r;
      j.vtW = sp<S>(f->vtW) + (size_t)(i + 1) * k * r;
      j.sT = f->sT.get() + (size_t)i * r;
      j.sW = f->sW.get() + (size_t)(i + 1) * r;
      j.K = sp<S>(f->Kd) + q * rr;
      j.E = sp<S>(f->Ed) + q * rr;
      j.Hinv = sp<S>(f->Hinv) + q * rr;
      j.cond = f->cond.get() + 2 * q;
      j.degenerate = f->degen.get() + q;
      jobs.push_back(j);
    }
    DevBuf<IfaceSetupJobT<S>> dj;
    upload(c, dj, jobs);
    launch_iface_setup_t<S>(c, dj.get(), ni, r, k);
    std::vector<double> hc(2 * ni);
    download(c, hc.data(), f->cond.get(), hc.size());
    for (int q = 0; q < ni; ++q) {
      const double ci = std::max(hc[2 * q], hc[2 * q + 1]);
      if (!(ci <= COND_LIMIT) && bad_i < 0) {
        bad_i = f->iface0 + q;
        bad_c = ci;
      }
      if (ci <= COND_LIMIT) mx = std::max(mx, ci);
    }
  }
  // every rank takes the same decision (first ill-conditioned interface in global order)
  {
    const std::vector<double> all = allgather_host(
        f, {bad_i >= 0 ? (double)bad_i : -1.0, bad_c, mx, f->rank_collapsed ? 1.0 : 0.0});
    bad_i = -1;
    for (size_t q = 0; q < all.size(); q += 4) {
      if (all[q] >= 0 && (bad_i < 0 || all[q] < bad_i)) {
        bad_i = (int)all[q];
        bad_c = all[q + 1];
      }
      mx = std::max(mx, all[q + 2]);
      f->rank_collapsed = f->rank_collapsed || all[q + 3] != 0.0;
    }
  }
  if (bad_i >= 0) {
    *bad_iface = bad_i;
    *bad_cond = bad_c;
    return false;
  }
  f->info.max_interface_cond = mx;
  // apply-time jobs
  const size_t scn = (size_t)Pg * r * MAX_RHS, msgn = (size_t)std::max(ni, 1) * 2 * r * MAX_RHS;
  f->scT.alloc(scn * w);
  f->scW.alloc(scn * w);
  f->iface_msg.alloc(msgn * w);
  LRS_CUDA(cudaMemsetAsync(f->scT.get(), 0, sizeof(S) * scn, c->stream));
  LRS_CUDA(cudaMemsetAsync(f->scW.get(), 0, sizeof(S) * scn, c->stream));
  LRS_CUDA(cudaMemsetAsync(f->iface_msg.get(), 0, sizeof(S) * msgn, c->stream));
  f->job_left = f->job_right = -1;
  {
    std::vector<IfaceApplyJobT<S>> jobs;
    for (int q = 0; q < ni; ++q) {
      const int i = f->iface0 + q;
      IfaceApplyJobT<S> j{};
      j.vtT = sp<S>(f->vtT) + (size_t)i * k * r;
      j.vtW = sp<S>(f->vtW) + (size_t)(i + 1) * k * r;
      j.sT = f->sT.get() + (size_t)i * r;
      j.sW = f->sW.get() + (size_t)(i + 1) * r;
      j.K = sp<S>(f->Kd) + q * rr;
      j.E = sp<S>(f->Ed) + q * rr;
      j.Hinv = sp<S>(f->Hinv) + q * rr;
      j.yb_row = goff(i) + gsize(i) - k;
      j.yt_row = goff(i + 1);
      j.scT = sp<S>(f->scT) + (size_t)i * r * MAX_RHS;
      j.scW = sp<S>(f->scW) + (size_t)(i + 1) * r * MAX_RHS;
      j.msg = sp<S>(f->iface_msg) + (size_t)q * 2 * r * MAX_RHS;
      j.has_left = (i >= p0 && i < p0 + P) ? 1 : 0;
      j.has_right = (i + 1 >= p0 && i + 1 < p0 + P) ? 1 : 0;
      if (!j.has_left) f->job_left = q;
      if (!j.has_right) f->job_right = q;
      jobs.push_back(j);
    }
    upload_raw(c, f->iface_jobs, jobs);
    // the same interfaces addressed in the compact reduced layout (LR-SPIKE-I / OTF):
    // bottom tip of partition i at row 2ki + k, top tip of partition i+1 at 2k(i+1)
    for (int q = 0; q < ni; ++q) {
      const int i = f->iface0 + q;
      jobs[q].yb_row = 2 * k * i + k;
      jobs[q].yt_row = 2 * k * (i + 1);
    }
    upload_raw(c, f->iface_jobs_red, jobs);
    f->iface_work.alloc(iface_work_doubles(std::max(ni, 1), r, k) * w);
  }
  LRS_CUDA(cudaStreamSynchronize(c->stream));
  return true;
}

template <class S>
bool build_lowrank(Fact* f, int r, int* bad_iface, double* bad_cond, const double* omega_dev) {
  Ctx* c = f->ctx;
  Mat* m = f->mat;
  const int Pg = f->Pg, p0 = f->p0, P = f->P;
  const int64_t n = f->n, k = f->k;
  const int os = f->os >= 0 ? f->os : (r + 1) / 2;
  const int l = r + os;
  constexpr int w = SW<S>;
  if (r < 1 || r > k) throw LrsError(LRS_ERR_PARAMETER, "randomized_spike_svd: 1 <= n_svd <= k");
  if (l > k) throw LrsError(LRS_ERR_PARAMETER, "randomized_spike_svd: n_svd + oversample <= k");
  if (f->passes < 2) throw LrsError(LRS_ERR_PARAMETER, "randomized_spike_svd: passes >= 2");
  if (l > 96) throw LrsError(LRS_ERR_PARAMETER, "n_svd + oversample > 96 not supported");
  f->r = r;
  f->l = l;
  const int L2 = 2 * l;
  DevBuf<double> Yb, Sb, Omb, Ztb, Rzb, Urb, Vrb, sig;
  Yb.alloc((size_t)n * L2 * w);
  Sb.alloc((size_t)n * L2 * w);
  Omb.alloc((size_t)Pg * 2 * k * l * w);
  Ztb.alloc((size_t)Pg * 2 * k * l * w);
  Rzb.alloc((size_t)Pg * 2 * l * l * w);
  Urb.alloc((size_t)Pg * 2 * l * l * w);
  Vrb.alloc((size_t)Pg * 2 * l * l * w);
  sig.alloc((size_t)Pg * 2 * l);
  S* Y = sp<S>(Yb);
  S* Sx = sp<S>(Sb);
  S* Om = sp<S>(Omb);
  S* Zt = sp<S>(Ztb);
  S* Rz = sp<S>(Rzb);
  S* Ur = sp<S>(Urb);
  S* Vr = sp<S>(Vrb);
  // local spikes: (global partition, side); partition g = p0 + local index
  std::vector<std::pair<int, int>> spk;
  for (int i = p0; i < p0 + P; ++i) {
    if (i < Pg - 1) spk.push_back({i, LRS_SIDE_T});
    if (i > 0) spk.push_back({i, LRS_SIDE_W});
  }
  auto slot = [&](int i, int side) { return (size_t)(2 * i + side); };
  auto goff = [&](int i) { return f->goff[i]; };
  auto gsize = [&](int i) { return f->goff[i + 1] - f->goff[i]; };
  // Omega from the shared counter-based generator, normally drawn by a
  // host thread while the band LU ran
  if (omega_dev) {
    // uploaded by omega_upload_task while the LU ran (the main stream already waits on it)
    const int64_t cnt = (int64_t)Pg * 2 * k * l;
    omega_expand_kernel<S><<<c->num_sms * 8, 256, 0, c->stream>>>(omega_dev, Om, cnt);
    LRS_LAUNCHED(c);
  } else {
    std::vector<double> h = make_omega(f->seed, Pg, p0, p0 + P, k, l);
    if constexpr (IsC<S>::value) {
      std::vector<double> hz(h.size() * 2, 0.0);
      for (size_t e = 0; e < h.size(); ++e) hz[2 * e] = h[e];
      h.swap(hz);
    }
    LRS_CUDA(cudaMemcpy(Om, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  }
  f->uT.alloc((size_t)n * r * w);
  f->uW.alloc((size_t)n * r * w);
  f->vtT.alloc((size_t)Pg * k * r * w);
  f->vtW.alloc((size_t)Pg * k * r * w);
  f->sT.alloc((size_t)Pg * r);
  f->sW.alloc((size_t)Pg * r);
  LRS_CUDA(cudaMemsetAsync(f->uT.get(), 0, sizeof(S) * n * r, c->stream));
  LRS_CUDA(cudaMemsetAsync(f->uW.get(), 0, sizeof(S) * n * r, c->stream));
  LRS_CUDA(cudaMemsetAsync(f->vtT.get(), 0, sizeof(S) * Pg * k * r, c->stream));
  LRS_CUDA(cudaMemsetAsync(f->vtW.get(), 0, sizeof(S) * Pg * k * r, c->stream));
  LRS_CUDA(cudaMemsetAsync(f->sT.get(), 0, sizeof(double) * Pg * r, c->stream));
  LRS_CUDA(cudaMemsetAsync(f->sW.get(), 0, sizeof(double) * Pg * r, c->stream));
  if (f->spike_mode == LRS_SPIKE_COUPLING) {
    coupling_spikes<S>(f, r, l, spk, Om, Y, Rz, Ur, Vr, sig.get());
  } else {
    auto ycol = [&](S* base, int i, int side) { return base + goff(i) + (int64_t)side * l * n; };
    // T_apply: Y = A_i^-1 pad(coupling X) for every spike, X = k x l blocks in src[slot]
    DevBuf<CoupleJobT<S>> cj;
    auto T_apply = [&](const S* src) {
      std::vector<CoupleJobT<S>> jobs;
      for (auto [i, side] : spk) {
        CoupleJobT<S> j{};
        if (side == LRS_SIDE_T) {
          j.r0 = goff(i) + gsize(i) - k;
          j.c0 = goff(i + 1);
        } else {
          j.r0 = goff(i);
          j.c0 = goff(i) - k;
        }
        j.b = k;
        j.dst0 = j.r0;
        j.X = src + slot(i, side) * k * l;
        j.ldx = k;
        j.out = Y + (int64_t)side * l * n;
        j.ldo = n;
        j.ncols = l;
        jobs.push_back(j);
      }
      LRS_CUDA(cudaMemsetAsync(Y, 0, sizeof(S) * n * L2, c->stream));
      upload(c, cj, jobs);
      launch_coupling_t<S>(c, m, false, cj.get(), (int)jobs.size(), k, l);
      dstage_t(f, Y, n, L2, false, -1);
    };
    // Tt_apply: Zt[slot] = coupling^H (A_i^-H Q)|tip, Q = columns of Y  (= T^H Q)
    auto Tt_apply = [&]() {
      copy_block(c, Sx, n, Y, n, n, L2);
      // real symmetric blocks: A_i^-T = A_i^-1, so the adjoint solve runs the (faster)
      // forward sweeps L, U instead of U^T, L^T
      dstage_t(f, Sx, n, L2, !(f->blocks_sym && !IsC<S>::value && !f->pivoted), -1);
      std::vector<CoupleJobT<S>> jobs;
      for (auto [i, side] : spk) {
        CoupleJobT<S> j{};
        if (side == LRS_SIDE_T) {  // B_i^H = A^H[off_{i+1} .., off_i+n_i-k ..]
          j.r0 = goff(i + 1);
          j.c0 = goff(i) + gsize(i) - k;
        } else {  // C_i^H = A^H[off_i - k .., off_i ..]
          j.r0 = goff(i) - k;
          j.c0 = goff(i);
        }
        j.b = k;
        j.dst0 = 0;
        j.X = Sx + j.c0 + (int64_t)side * l * n;
        j.ldx = n;
        j.out = Zt + slot(i, side) * k * l;
        j.ldo = k;
        j.ncols = l;
        jobs.push_back(j);
      }
      upload(c, cj, jobs);
      launch_coupling_t<S>(c, m, true, cj.get(), (int)jobs.size(), k, l);
    };
    DevBuf<QrJobT<S>> qj;
    auto orth_Y = [&]() {
      std::vector<QrJobT<S>> jobs;
      int64_t mm = n;
      for (auto [i, side] : spk) {
        jobs.push_back(QrJobT<S>{ycol(Y, i, side), gsize(i), n, nullptr});
        mm = std::min(mm, gsize(i));
      }
      upload(c, qj, jobs);
      launch_householder_qr_t<S>(c, qj.get(), (int)jobs.size(), l, mm);
    };
    auto orth_Zt = [&](bool keepR) {
      std::vector<QrJobT<S>> jobs;
      for (auto [i, side] : spk)
        jobs.push_back(QrJobT<S>{Zt + slot(i, side) * k * l, k, k,
                                 keepR ? Rz + slot(i, side) * l * l : nullptr});
      upload(c, qj, jobs);
      launch_householder_qr_t<S>(c, qj.get(), (int)jobs.size(), l, k);
    };

    T_apply(Om);
    orth_Y();
    for (int pi = 0; pi < (f->passes - 2) / 2; ++pi) {
      Tt_apply();
      orth_Zt(false);
      T_apply(Zt);
      orth_Y();
    }
    Tt_apply();          // Zt = (Q^H T)^H, k x l
    orth_Zt(true);       // Zt = Q_z R_z
    {
      std::vector<SvdJobT<S>> jobs;
      for (auto [i, side] : spk) {
        const size_t s = slot(i, side);
        jobs.push_back(SvdJobT<S>{Rz + s * l * l, Vr + s * l * l, Ur + s * l * l, sig.get() + s * l});
      }
      DevBuf<SvdJobT<S>> sj;
      upload(c, sj, jobs);
      launch_jacobi_svd_t<S>(c, sj.get(), (int)jobs.size(), l);
      // Z = V_R S (Q_z U_R)^H  =>  u = Q V_R[:, :r],  v^T = conj(Q_z U_R[:, :r])
      std::vector<GemmJobT<S>> gu, gv;
      std::vector<SigmaJob> sjobs;
      int64_t maxm = 0;
      for (auto [i, side] : spk) {
        const size_t s = slot(i, side);
        S* ubuf = side == LRS_SIDE_T ? sp<S>(f->uT) : sp<S>(f->uW);
        S* vbuf = side == LRS_SIDE_T ? sp<S>(f->vtT) : sp<S>(f->vtW);
        double* sbuf = side == LRS_SIDE_T ? f->sT.get() : f->sW.get();
        gu.push_back(GemmJobT<S>{ycol(Y, i, side), n, Vr + s * l * l, l, ubuf + goff(i), n,
                                 gsize(i), r, l, 0});
        gv.push_back(GemmJobT<S>{Zt + s * k * l, k, Ur + s * l * l, l, vbuf + (size_t)i * k * r, k,
                                 k, r, l, IsC<S>::value ? 1 : 0});
        sjobs.push_back(SigmaJob{sig.get() + s * l, sbuf + (size_t)i * r});
        maxm = std::max(maxm, gsize(i));
      }
      DevBuf<GemmJobT<S>> dgu, dgv;
      upload(c, dgu, gu);
      upload(c, dgv, gv);
      launch_small_gemm_t<S>(c, dgu.get(), (int)gu.size(), maxm, r);
      launch_small_gemm_t<S>(c, dgv.get(), (int)gv.size(), k, r);
      DevBuf<SigmaJob> dsj;
      upload(c, dsj, sjobs);
      DevBuf<int> flag;
      flag.alloc(1);
      LRS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), c->stream));
      launch_sigma_trunc(c, dsj.get(), (int)sjobs.size(), r, flag.get());
      int hflag = 0;
      download(c, &hflag, flag.get(), 1);
      f->rank_collapsed = hflag != 0;
    }
  }  // spike_mode
  // C5: ship the T side of the last local partition right and the W side of the first
  // local partition left: [u tip (k x r) | v^T (k x r) | sigma (r, real)]
  if (f->dist) {
    const int64_t kr = k * r, cnt = 2 * kr * w + r;  // doubles
    DevBuf<double> buf;
    buf.alloc((size_t)cnt * 4);
    double* s_next = buf.get();
    double* r_prev = s_next + cnt;
    double* s_prev = r_prev + cnt;
    double* r_next = s_prev + cnt;
    auto U = [](double* b) { return reinterpret_cast<S*>(b); };
    auto pack = [&](double* dst, const S* ubuf, int64_t urow, const S* vbuf, const double* sbuf,
                    int i) {
      copy_block(c, U(dst), k, ubuf + urow, n, k, r);
      LRS_CUDA(cudaMemcpyAsync(U(dst) + kr, vbuf + (size_t)i * kr, sizeof(S) * kr,
                               cudaMemcpyDeviceToDevice, c->stream));
      LRS_CUDA(cudaMemcpyAsync(dst + 2 * kr * w, sbuf + (size_t)i * r, sizeof(double) * r,
                               cudaMemcpyDeviceToDevice, c->stream));
    };
    auto unpack = [&](const double* src, S* ubuf, int64_t urow, S* vbuf, double* sbuf, int i) {
      copy_block(c, ubuf + urow, n, reinterpret_cast<const S*>(src), k, k, r);
      LRS_CUDA(cudaMemcpyAsync(vbuf + (size_t)i * kr, reinterpret_cast<const S*>(src) + kr,
                               sizeof(S) * kr, cudaMemcpyDeviceToDevice, c->stream));
      LRS_CUDA(cudaMemcpyAsync(sbuf + (size_t)i * r, src + 2 * kr * w, sizeof(double) * r,
                               cudaMemcpyDeviceToDevice, c->stream));
    };
    const int iR = p0 + P - 1;  // T side, to the right neighbour (if any)
    if (iR < Pg - 1) pack(s_next, sp<S>(f->uT), goff(iR + 1) - k, sp<S>(f->vtT), f->sT.get(), iR);
    if (p0 > 0) pack(s_prev, sp<S>(f->uW), goff(p0), sp<S>(f->vtW), f->sW.get(), p0);
    neighbor_exchange(f, s_next, r_prev, s_prev, r_next, cnt);
    if (p0 > 0)  // T side of partition p0 - 1
      unpack(r_prev, sp<S>(f->uT), goff(p0) - k, sp<S>(f->vtT), f->sT.get(), p0 - 1);
    if (iR < Pg - 1)  // W side of partition iR + 1
      unpack(r_next, sp<S>(f->uW), goff(iR + 1), sp<S>(f->vtW), f->sW.get(), iR + 1);
  }
  return finish_interfaces<S>(f, r, bad_iface, bad_cond);
}

}  // namespace

void shard_plan(int64_t P, int size, int rank, int64_t* p_lo, int64_t* p_hi) {
  *p_lo = (int64_t)rank * P / size;
  *p_hi = (int64_t)(rank + 1) * P / size;
}

void dstage(Fact* f, void* x, int64_t ld, int nrhs, bool adjoint, int p_only) {
  if (f->scalar == LRS_C128) dstage_t(f, static_cast<zc*>(x), ld, nrhs, adjoint, p_only);
  else dstage_t(f, static_cast<double*>(x), ld, nrhs, adjoint, p_only);
}


// ------------------------------------------------------------------------------------
// factorize
// ------------------------------------------------------------------------------------
Fact* factorize(Ctx* c, Mat* m, const lrs_solver_cfg& cfg, const lrs_comm* comm) {
  std::unique_ptr<Fact> f(new Fact());
  f->ctx = c;
  f->mat = m;
  f->scalar = m->scalar;
  f->sw = m->scalar == LRS_C128 ? 2 : 1;
  const bool cplx = f->scalar == LRS_C128;
  f->variant = cfg.variant;
  if (cfg.variant != LRS_VARIANT_T && cfg.variant != LRS_VARIANT_BJ &&
      cfg.variant != LRS_VARIANT_I && cfg.variant != LRS_VARIANT_OTF)
    throw LrsError(LRS_ERR_PARAMETER, "unknown variant");
  f->inner_tol = cfg.inner_tol > 0 ? cfg.inner_tol : 1e-12;
  f->inner_max_iters = cfg.inner_max_iters > 0 ? cfg.inner_max_iters : 200;
  f->otf_tol = cfg.otf_tol > 0 ? cfg.otf_tol : 1e-8;
  f->otf_max_iters = cfg.otf_max_iters > 0 ? cfg.otf_max_iters : 500;
  f->otf_escalations = cfg.otf_escalations >= 0 ? cfg.otf_escalations : 4;
  if (cfg.p < 1) throw LrsError(LRS_ERR_PARAMETER, "p >= 1 required");
  if (cfg.n_svd < 0) throw LrsError(LRS_ERR_PARAMETER, "n_svd >= 0 required");
  if (comm && comm->size > 1) {
    if (!comm->allgather || !comm->sendrecv)
      throw LrsError(LRS_ERR_PARAMETER, "lrs_comm needs allgather and sendrecv callbacks");
    if (comm->rank < 0 || comm->rank >= comm->size)
      throw LrsError(LRS_ERR_PARAMETER, "lrs_comm rank out of range");
    if (cfg.p < comm->size) throw LrsError(LRS_ERR_PARAMETER, "p must be >= the number of GPUs");
    f->dist = true;
    f->comm = *comm;
  }
  const int G = f->nranks(), rank = f->rank();
  const int w = f->sw;
  f->Pg = (int)cfg.p;
  f->n = m->n;
  f->k = cfg.k > 0 ? cfg.k : m->k;
  f->kl = m->kl;
  f->ku = m->ku;
  f->passes = cfg.passes > 0 ? cfg.passes : 2;
  f->seed = cfg.seed;
  f->os = (int)cfg.oversample;
  if (cfg.spike_mode != LRS_SPIKE_SVD && cfg.spike_mode != LRS_SPIKE_COUPLING)
    throw LrsError(LRS_ERR_PARAMETER, "spike_mode must be LRS_SPIKE_SVD or LRS_SPIKE_COUPLING");
  f->spike_mode = cfg.spike_mode;
  // global layout and this rank's shard
  {
    const int64_t Pg = f->Pg, n = f->n;
    f->goff.assign(Pg + 1, 0);
    int64_t mn = n;
    for (int64_t i = 0; i < Pg; ++i) {
      const int64_t s = n / Pg + (i < n % Pg ? 1 : 0);
      f->goff[i + 1] = f->goff[i] + s;
      mn = std::min(mn, s);
    }
    if (mn <= f->k)
      throw LrsError(LRS_ERR_LAYOUT, "layout infeasible: need n >= p*(k+1) = " +
                                         std::to_string(Pg * (f->k + 1)));
    int64_t plo, phi;
    shard_plan(Pg, G, rank, &plo, &phi);
    f->p0 = (int)plo;
    f->P = (int)(phi - plo);
    f->row_lo = f->goff[plo];
    f->row_hi = f->goff[phi];
    f->off.resize(f->P);
    f->size.resize(f->P);
    for (int i = 0; i < f->P; ++i) {
      f->off[i] = f->goff[plo + i];
      f->size[i] = f->goff[plo + i + 1] - f->goff[plo + i];
    }
    f->rank_pl.resize(G);
    f->pl_max = 0;
    for (int q = 0; q < G; ++q) {
      int64_t a, b;
      shard_plan(Pg, G, q, &a, &b);
      f->rank_pl[q] = (int)(b - a);
      f->pl_max = std::max(f->pl_max, f->rank_pl[q]);
    }
  }
  const int P = f->P;
  f->T.resize(P);
  f->tbase.resize(P);
  f->fbase.resize(P);
  f->Tmax = 0;
  int Tmax_all = 0;
  for (int i = 0; i < f->Pg; ++i)
    Tmax_all = std::max<int>(Tmax_all, (int)((f->goff[i + 1] - f->goff[i] + NB - 1) / NB));
  for (int i = 0; i < P; ++i) {
    f->T[i] = (int)((f->size[i] + NB - 1) / NB);
    f->Tmax = std::max(f->Tmax, f->T[i]);
  }
  upload(c, f->d_off, f->off);
  upload(c, f->d_size, f->size);
  upload(c, f->d_T, f->T);
  upload(c, f->d_goff, f->goff);
  upload(c, f->d_rank_pl, f->rank_pl);
  // tile storage for an upper band of ku_eff (ku, or ku + kl with row interchanges); band
  // widths in tiles from the global block sizes, identical on every rank
  auto setup_tiles = [&](int64_t ku_eff) {
    f->wl = std::min((int)((f->kl + NB - 1) / NB), std::max(0, Tmax_all - 1));
    f->wu = std::min((int)((ku_eff + NB - 1) / NB), std::max(0, Tmax_all - 1));
    f->W = f->wl + f->wu + 1;
    int64_t tb = 0, fb = 0;
    for (int i = 0; i < P; ++i) {
      f->tbase[i] = tb;
      f->fbase[i] = fb;
      tb += (int64_t)f->T[i] * f->W;
      fb += f->T[i];
    }
    f->total_tiles = tb;
    f->total_rowtiles = fb;
    upload(c, f->d_tbase, f->tbase);
    upload(c, f->d_fbase, f->fbase);
    f->tiles.reset();
    f->tiles.alloc((size_t)tb * TILE_ELEMS * w);
    f->flags.alloc((size_t)fb * SOLVE_GROUPS);
    f->mbox.alloc((size_t)fb * 2 * NB);
    f->ticket.alloc(1);
    f->status.alloc(2 * P);
    f->bad.alloc(1);
    LRS_CUDA(cudaMemsetAsync(f->tiles.get(), 0, sizeof(double) * tb * TILE_ELEMS * w, c->stream));
    LRS_CUDA(cudaMemsetAsync(f->flags.get(), 0, sizeof(unsigned) * fb * SOLVE_GROUPS, c->stream));
    LRS_CUDA(cudaMemsetAsync(f->mbox.get(), 0, sizeof(unsigned long long) * fb * 2 * NB, c->stream));
    LRS_CUDA(cudaMemsetAsync(f->status.get(), 0x7f, sizeof(int) * 2 * P, c->stream));
    LRS_CUDA(cudaMemsetAsync(f->bad.get(), 0xff, sizeof(unsigned long long), c->stream));
  };
  setup_tiles(f->ku);
  // deterministic reduction chunks, partition aligned
  {
    const int64_t CH = KRYLOV_CHUNK;
    f->chunk_start.clear();
    f->part_first.assign(P + 1, 0);
    for (int i = 0; i < P; ++i) {
      f->part_first[i] = (int)f->chunk_start.size();
      for (int64_t r0 = 0; r0 < f->size[i]; r0 += CH) f->chunk_start.push_back(f->off[i] + r0);
    }
    f->part_first[P] = (int)f->chunk_start.size();
    f->chunk_start.push_back(f->row_hi);
    upload(c, f->d_chunks, f->chunk_start);
    upload(c, f->d_part_first, f->part_first);
    // the compact reduced space (2k rows per partition)
    const int64_t k2 = 2 * f->k;
    f->ldr = k2 * f->Pg;
    f->rchunk_start.clear();
    f->rpart_first.assign(P + 1, 0);
    for (int i = 0; i < P; ++i) {
      f->rpart_first[i] = (int)f->rchunk_start.size();
      for (int64_t r0 = 0; r0 < k2; r0 += CH) f->rchunk_start.push_back(k2 * (f->p0 + i) + r0);
    }
    f->rpart_first[P] = (int)f->rchunk_start.size();
    f->rchunk_start.push_back(k2 * (f->p0 + P));
    upload(c, f->d_rchunks, f->rchunk_start);
    upload(c, f->d_rpart_first, f->rpart_first);
    const size_t nch = std::max(f->chunk_start.size(), f->rchunk_start.size()) - 1;
    f->partial.alloc(nch * 64 * MAX_RHS * w);
    f->persum.alloc((size_t)f->pl_max * 64 * MAX_RHS * w);
    f->gather.alloc((size_t)G * f->pl_max * 64 * MAX_RHS * w);
    f->dotout.alloc(64 * MAX_RHS * w);
    f->xch.alloc((size_t)4 * std::max<int64_t>(1, std::max(m->k, f->k)) * MAX_RHS * w);
  }
  cudaEvent_t e0, e1, e2, e3;
  LRS_CUDA(cudaEventCreate(&e0));
  LRS_CUDA(cudaEventCreate(&e1));
  LRS_CUDA(cudaEventCreate(&e2));
  LRS_CUDA(cudaEventCreate(&e3));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  };
  cudaEvent_t evs[4] = {e0, e1, e2, e3};
  EvGuard eg{evs};
  LRS_CUDA(cudaEventRecord(e0, c->stream));
  BandGeom g = f->geom();
  if (cplx)
    launch_extract_tiles_z(c, m, g, sp<zc>(f->tiles), f->k, f->row_lo, f->row_hi, f->bad.get());
  else
    launch_extract_tiles(c, m, g, f->tiles.get(), f->k, f->row_lo, f->row_hi, f->bad.get());
  {
    unsigned long long hb = 0;
    download(c, &hb, f->bad.get(), 1);
    // agree on the first offending entry over all ranks (row-major order)
    const std::vector<double> all = allgather_host(f.get(), {hb == ~0ull ? -1.0 : (double)hb});
    double first = -1.0;
    for (double v : all)
      if (v >= 0 && (first < 0 || v < first)) first = v;
    if (first >= 0) {
      const unsigned long long hv = (unsigned long long)first;
      LrsError e(LRS_ERR_NOT_BLOCK_TRIDIAGONAL,
                 "nonzero (" + std::to_string(hv / f->n) + "," + std::to_string(hv % f->n) +
                     ") outside the block-tridiagonal pattern; increase k or decrease p");
      e.row = (int64_t)(hv / f->n);
      e.col = (int64_t)(hv % f->n);
      throw e;
    }
  }
  // structurally nonzero couplings? (LR-SPIKE-OTF skips the reduced solve without any)
  {
    DevBuf<int> flag;
    flag.alloc(1);
    LRS_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), c->stream));
    launch_coupling_present(c, m, g, f->row_lo, f->row_hi, flag.get());
    int hf = 0;
    download(c, &hf, flag.get(), 1);
    double any_c = hf;
    for (double v : allgather_host(f.get(), {(double)hf})) any_c = std::max(any_c, v);
    f->coupled = any_c > 0 && f->Pg > 1;
  }
  // the host draws Omega for the spike SVDs while the GPU runs the band LU
  // a host thread draws Omega for the spike SVDs into page-locked memory and uploads it on
  // the copy stream while the GPU runs the band LU
  // (destruction order on an early exit: the future joins the host thread, the guard drains
  // the copy stream, and only then omega_dev goes back to the pool)
  DevBuf<double> omega_dev;
  struct CopyGuard {
    Ctx* c;
    cudaEvent_t ev = nullptr;  // recorded on the main stream when omega_dev was allocated
    ~CopyGuard() {
      cudaStreamSynchronize(c->stream_copy);
      if (ev) c->ev_pool.push_back(ev);
    }
  } omega_guard{c};
  std::future<bool> omega_future;
  {
    const int r0 = (int)cfg.n_svd;
    const int l0 = r0 + (cfg.oversample >= 0 ? (int)cfg.oversample : (r0 + 1) / 2);
    if ((f->variant == LRS_VARIANT_T || f->variant == LRS_VARIANT_I ||
         f->variant == LRS_VARIANT_OTF) && f->Pg > 1 && r0 >= 1 && l0 <= f->k) {
      omega_dev.alloc((size_t)f->Pg * 2 * f->k * l0);
      omega_guard.ev = c->take_event();
      LRS_CUDA(cudaEventRecord(omega_guard.ev, c->stream));
      omega_future = std::async(std::launch::async, omega_upload_task, c, omega_dev.get(),
                                omega_guard.ev, f->seed, f->Pg, f->p0, f->p0 + P, f->k, l0);
    }
  }
  if (cplx)
    f->lu_int8 = launch_band_lu_z(c, g, sp<zc>(f->tiles), f->Tmax, f->status.get(),
                                  mat_is_symmetric(c, m), &f->lu_sym);
  else
    f->lu_int8 = launch_band_lu(c, g, f->tiles.get(), f->Tmax, f->status.get(),
                                mat_is_symmetric(c, m), &f->lu_sym);
  {
    const char* e = std::getenv("LRS_LU_SYM");
    f->blocks_sym = mat_is_symmetric(c, m) && !(e && e[0] == '0');
  }
  // first (global block, column) needing a row interchange / holding an exact zero pivot,
  // agreed over all ranks
  auto first_problem = [&](int which) {
    std::vector<int> st(2 * P);
    download(c, st.data(), f->status.get(), st.size());
    double blk = -1, col = 0;
    for (int i = 0; i < P && blk < 0; ++i)
      if (st[2 * i + which] != 0x7f7f7f7f) {
        blk = f->p0 + i;
        col = st[2 * i + which];
      }
    std::pair<int, int64_t> out{-1, 0};
    const std::vector<double> all = allgather_host(f.get(), {blk, col});
    for (size_t q = 0; q < all.size(); q += 2)
      if (all[q] >= 0) {
        out = {(int)all[q], (int64_t)all[q + 1]};
        break;
      }
    return out;
  };
  if (first_problem(0).first >= 0) {
    // dgbtrf would interchange rows: redo the blocks with partial pivoting (upper band
    // widened by kl for the fill of the interchanges)
    setup_tiles(f->ku + f->kl);
    g = f->geom();
    if (cplx)
      launch_extract_tiles_z(c, m, g, sp<zc>(f->tiles), f->k, f->row_lo, f->row_hi, f->bad.get());
    else
      launch_extract_tiles(c, m, g, f->tiles.get(), f->k, f->row_lo, f->row_hi, f->bad.get());
    f->pivoted = true;
    f->ipiv.alloc((size_t)f->total_rowtiles * NB);
    f->perm.alloc(piv_perm_ints(f->total_rowtiles));
    if (cplx)
      launch_band_lu_piv_z(c, g, sp<zc>(f->tiles), f->Tmax, f->status.get(), f->ipiv.get(),
                           f->perm.get());
    else
      launch_band_lu_piv(c, g, f->tiles.get(), f->Tmax, f->status.get(), f->ipiv.get(),
                         f->perm.get());
  }
  LRS_CUDA(cudaEventRecord(e1, c->stream));
  if (cfg.factor_fp32) {
    if (cplx || f->pivoted)
      throw LrsError(LRS_ERR_NOT_IMPLEMENTED,
                     "FP32 factors: real blocks without row interchanges only");
    // slot (I, J - I + wl) of row tile I lies inside its block for 0 <= J < T; the FP32
    // copy stores those densely (c3 at P = 64: 66% of the 147-slot rows of a 108-tile block)
    std::vector<int> idx((size_t)f->total_tiles, -1);
    int64_t cnt = 0;
    for (int p = 0; p < P; ++p)
      for (int I = 0; I < f->T[p]; ++I)
        for (int J = std::max(0, I - f->wl); J <= std::min(f->T[p] - 1, I + f->wu); ++J)
          idx[(size_t)(f->tbase[p] + (int64_t)I * f->W + (J - I + f->wl))] = (int)cnt++;
    if (cnt >= (int64_t(1) << 31)) throw LrsError(LRS_ERR_DIMENSION, "too many factor tiles");
    upload(c, f->t32_idx, idx);
    f->tiles32_count = cnt;
    f->tiles32.alloc((size_t)cnt * TILE_ELEMS);
    launch_tiles_to_fp32(c, f->tiles.get(), f->tiles32.get(), f->t32_idx.get(), f->total_tiles);
    f->fp32 = true;
  }
  {
    const auto pr = first_problem(1);
    if (pr.first >= 0) {
      LrsError e(LRS_ERR_SINGULAR_BLOCK, "exact zero pivot in column " + std::to_string(pr.second) +
                                             " of block " + std::to_string(pr.first));
      e.column = pr.second;
      throw e;
    }
  }
  // spikes + truncated preconditioner, with the r-halving retry
  const bool spiked = f->variant == LRS_VARIANT_T || f->variant == LRS_VARIANT_I ||
                      f->variant == LRS_VARIANT_OTF;
  int r = (spiked && f->Pg > 1) ? (int)cfg.n_svd : 0;
  f->r = 0;
  f->l = 0;
  if (r > 0) {
    for (int attempt = 0;; ++attempt) {
      int bi = -1;
      double bc = 0.0;
      c->in_setup = true;
      bool ok;
      try {
        const double* pre = nullptr;
        if (attempt == 0 && omega_future.valid() && omega_future.get()) {
          LRS_CUDA(cudaStreamWaitEvent(c->stream, c->ev_omega, 0));
          pre = omega_dev.get();
        }
        ok = cplx ? build_lowrank<zc>(f.get(), r, &bi, &bc, pre)
                  : build_lowrank<double>(f.get(), r, &bi, &bc, pre);
      } catch (...) {
        c->in_setup = false;
        throw;
      }
      c->in_setup = false;
      if (ok) break;
      if (attempt == 1 || r / 2 < 1) {
        LrsError e(LRS_ERR_ILL_CONDITIONED_INTERFACE,
                   "interface " + std::to_string(bi) + " ill-conditioned (cond " +
                       std::to_string(bc) + ")");
        e.iface = bi;
        e.cond = bc;
        throw e;
      }
      r /= 2;
    }
  }
  LRS_CUDA(cudaEventRecord(e2, c->stream));
  LRS_CUDA(cudaEventSynchronize(e2));
  // info
  lrs_fact_info& in = f->info;
  in.n = f->n;
  in.p = f->Pg;
  in.k = f->k;
  in.n_svd = f->r;
  in.l = f->l;
  in.kl = f->kl;
  in.ku = f->ku;
  in.nb = NB;
  in.wl = f->wl;
  in.wu = f->wu;
  in.factor_bytes = f->total_tiles * TILE_ELEMS * (int64_t)sizeof(double) * w +
                    (f->fp32 ? f->tiles32_count * TILE_ELEMS * (int64_t)sizeof(float) : 0);
  in.rank_collapsed = f->rank_collapsed;
  in.variant = f->variant;
  // steps per bulk update launch: 4 (INT8 quads), 2 (pairs), 0 (single steps)
  in.lu_pairs = f->pivoted ? 0 : (f->lu_int8 ? f->lu_int8 : (!cplx && lu_real_pairs(g) ? 2 : 0));
  in.pivoted = f->pivoted ? 1 : 0;
  in.lu_int8 = f->lu_int8 ? 1 : 0;
  in.lu_sym = (f->lu_sym && !f->pivoted) ? 1 : 0;
  in.t_lu = elapsed_ms(e0, e1) * 1e-3;
  in.t_spikes = elapsed_ms(e1, e2) * 1e-3;
  in.t_precond = 0.0;
  in.t_factorize = elapsed_ms(e0, e2) * 1e-3;
  if (in.max_interface_cond == 0.0) in.max_interface_cond = 1.0;
  // algorithmic work of THIS shard: no-fill band LU flops (x4 for
  // complex arithmetic), apply bytes
  double flops = 0.0, fbytes = 0.0;
  for (int i = 0; i < P; ++i) {
    const int64_t ni = f->size[i];
    for (int64_t j = 0; j < ni; ++j) {
      const double rem = (double)(ni - 1 - j);
      const double a = std::min<double>((double)f->kl, rem), b = std::min<double>((double)f->ku, rem);
      flops += a + 2.0 * a * b;
      fbytes += a + 1.0 + b;
    }
  }
  const double nl = (double)(f->row_hi - f->row_lo);
  in.lu_flops = (int64_t)(flops * (cplx ? 4.0 : 1.0));
  // FP32 factors: the off-diagonal band entries at 4 bytes, the diagonal tiles at 8
  double diag_entries = 0.0;
  for (int i = 0; i < P; ++i) diag_entries += (double)f->T[i] * NB * NB;
  diag_entries = std::min(diag_entries, fbytes);
  in.apply_bytes = f->fp32 ? (int64_t)(4.0 * (fbytes - diag_entries) + 8.0 * diag_entries +
                                       8.0 * (2.0 * nl + 2.0 * nl * f->r))
                           : (int64_t)(8.0 * w * (fbytes + 2.0 * nl + 2.0 * nl * f->r));
  return f.release();
}

// ------------------------------------------------------------------------------------
// Krylov drivers (mirror the checker's bicgstab / gmres); vector work on the local rows
// ------------------------------------------------------------------------------------
namespace {

// A Krylov space: full-length blocks with leading dimension n, this GPU's rows
// [lo, lo + nl), partition-aligned reduction chunks, and the operator / preconditioner.
// The outer solve works in the n-layout (A = the CSR, M = the preconditioner); the
// LR-SPIKE-I inner solve and the LR-SPIKE-OTF reduced solve in the compact reduced space.
template <class S>
struct Work {
  using H = HT<S>;
  Fact* f;
  int64_t n;       // full length (ld of every block)
  int64_t lo, nl;  // local rows [lo, lo + nl)
  Chunks ch;       // deterministic reduction chunks of the space
  int nr;
  lrs_report* rep;
  std::vector<double> hist;
  double* hbuf = nullptr;  // pinned landing buffer of the dot products (Ctx-owned)
  std::function<void(const S*, S*)> Mf;            // out = M^-1 in
  std::function<void(S*, S*)> Af;                  // out = A in (halo rows of in may be written)
  std::function<void(const S*, S*, S*)> Rf;        // out = b - A x
  std::function<void(S*, S*, const S*)> AfD;       // out = A in + chunk partials of [X^H out, out^H out]
  void init() { hbuf = f->ctx->dots_host; }
  Ctx* c() const { return f->ctx; }
  S* dotout() const { return sp<S>(f->dotout); }
  // out[q*nr + j] = X_q[:, j]^H Y[:, j] over ALL rows (partition-ordered, any GPU count)
  void dots(const S* X, int64_t strideX, int nvec, const S* Y, H* out) {
    launch_multidot_partition_t<S>(c(), ch, X, n, strideX, nvec, Y, n, nr,
                                   sp<S>(f->partial), sp<S>(f->persum));
    dots_finish(nvec, out);
  }
  // out = A in and [X^H out, out^H out] (BiCGStab's t = A shat with t^H s, t^H t): the
  // fused SpMV-dot kernel where the operator is the CSR (AfD set), else SpMV + dots
  void Aop_dots2(S* in, S* out, const S* X, H* res) {
    if (!AfD) {
      Aop(in, out);
      return dots(X, (int64_t)(out - X), 2, out, res);
    }
    AfD(in, out, X);
    rep->matvecs++;
    launch_multidot_persum(c(), ch, 2 * nr * SW<S>, f->partial.get(), f->persum.get());
    dots_finish(2, res);
  }
  // dots without the host round trip: the totals land in pinned slot `slot` when the stream
  // gets there (GMRES reads the three CGS2 results after ONE synchronization per step)
  static constexpr size_t SLOT = 64 * MAX_RHS * 2;  // doubles per slot
  void dots_enqueue(const S* X, int64_t strideX, int nvec, const S* Y, int slot) {
    launch_multidot_partition_t<S>(c(), ch, X, n, strideX, nvec, Y, n, nr, sp<S>(f->partial),
                                   sp<S>(f->persum));
    dots_total(nvec, hbuf + slot * SLOT);
  }
  void dots_wait() {
    LRS_CUDA(cudaStreamSynchronize(c()->stream));
    ++f->scalar_syncs;
  }
  void dots_read(int nvec, int slot, H* out) const {
    std::memcpy(static_cast<void*>(out), hbuf + slot * SLOT, sizeof(double) * nvec * nr * SW<S>);
  }
  // per-partition sums -> global totals (dotout) -> async copy to `host`
  void dots_total(int nvec, double* host) {
    const int nout = nvec * nr * SW<S>;  // doubles
    if (f->dist) {
      if (!f->comm.stream_ordered) {
        LRS_CUDA(cudaStreamSynchronize(c()->stream));
        ++f->comm_syncs;
      }
      ++f->comm_calls;
      comm_rc(f->comm.allgather(f->comm.user, f->persum.get(), f->gather.get(),
                                (int64_t)f->pl_max * nout),
              "allgather");
      launch_partition_total(c(), f->gather.get(), f->d_rank_pl.get(), f->comm.size, f->pl_max,
                             nout, f->dotout.get());
    } else {
      launch_partition_total(c(), f->persum.get(), f->d_rank_pl.get(), 1, f->P, nout,
                             f->dotout.get());
    }
    LRS_CUDA(cudaMemcpyAsync(host, f->dotout.get(), sizeof(double) * nout, cudaMemcpyDeviceToHost,
                             c()->stream));
  }
  // per-partition sums (persum) -> global partition-ordered totals -> host
  void dots_finish(int nvec, H* out) {
    dots_total(nvec, hbuf);
    dots_wait();
    dots_read(nvec, 0, out);
  }
  void norms(const S* X, double* out) {
    std::vector<H> d(nr);
    dots(X, 0, 1, X, d.data());
    for (int j = 0; j < nr; ++j) out[j] = std::sqrt(hreal(d[j]));
  }
  void M(const S* in, S* out) {
    Mf(in, out);
    rep->precond_applications++;
  }
  void Aop(S* in, S* out) {
    Af(in, out);
    rep->matvecs++;
  }
  void resid(const S* b, S* x, S* out) {  // out = b - A x
    Rf(b, x, out);
    rep->matvecs++;
  }
  void axpby(int op, const ColScalT<S>& a, const ColScalT<S>& b, const ColScal& act, S* X,
             const S* Y, const S* Z, S* Wv) {
    launch_axpby_cols_t<S>(c(), nl, nr, op, a, b, act, X ? X + lo : nullptr, n,
                           Y ? Y + lo : nullptr, n, Z ? Z + lo : nullptr, n,
                           Wv ? Wv + lo : nullptr, n);
  }
  void copy(S* dst, const S* src) { copy_block(c(), dst + lo, n, src + lo, n, nl, nr); }
  void zero(S* dst) {
    for (int j = 0; j < nr; ++j)
      LRS_CUDA(cudaMemsetAsync(dst + lo + (int64_t)j * n, 0, sizeof(S) * nl, c()->stream));
  }
  void push(double v) { hist.push_back(v); }
};

template <class S>
ColScalT<S> cs_fill(const std::vector<HT<S>>& v) {
  ColScalT<S> s{};
  for (size_t j = 0; j < v.size() && j < MAX_RHS; ++j) s.v[j] = to_dev<S>(v[j]);
  return s;
}
ColScal cs_mask(const std::vector<bool>& v) {
  ColScal s{};
  for (size_t j = 0; j < v.size() && j < MAX_RHS; ++j) s.v[j] = v[j] ? 1.0 : 0.0;
  return s;
}
bool any(const std::vector<bool>& v) {
  for (bool b : v)
    if (b) return true;
  return false;
}

template <class S>
void run_bicgstab(Work<S>& w, const S* b, S* x, const lrs_iter_cfg& cfg, bool has_x0,
                  std::vector<double>& iters, std::vector<bool>& conv, std::vector<bool>& brk) {
  using H = HT<S>;
  const int nr = w.nr;
  const int64_t n = w.n;
  const size_t blk = (size_t)n * nr;
  DevBuf<S> buf;
  buf.alloc(blk * 9);
  S* r = buf.get();
  S* rhat = r + blk;
  S* p = rhat + blk;
  S* v = p + blk;
  S* s = v + blk;
  S* t = s + blk;
  S* phat = t + blk;
  S* shat = phat + blk;
  S* tmp = shat + blk;
  const ColScalT<S> none{};
  std::vector<double> bn(nr), bns(nr), tmpv(nr), tmpv2(nr);
  w.norms(b, bn.data());
  for (int j = 0; j < nr; ++j) bns[j] = bn[j] > 0 ? bn[j] : 1.0;
  if (has_x0) {
    w.resid(b, x, r);
  } else {
    w.zero(x);
    w.copy(r, b);
  }
  w.norms(r, tmpv.data());
  double mx = 0;
  conv.assign(nr, false);
  brk.assign(nr, false);
  iters.assign(nr, 0.0);
  for (int j = 0; j < nr; ++j) {
    conv[j] = tmpv[j] / bns[j] <= cfg.tol || bn[j] == 0.0;
    mx = std::max(mx, tmpv[j] / bns[j]);
  }
  w.push(mx);
  w.copy(rhat, r);
  std::vector<H> rho_prev(nr, H(1.0)), alpha(nr, H(1.0)), omega(nr, H(1.0)), rho(nr), rv(nr);
  w.zero(p);
  w.zero(v);
  const bool trace = std::getenv("LRS_TRACE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  // rho = rhat^H r of the next iteration comes with the norm of the new r (one reduction,
  // one host round trip: r and rhat sit one block apart)
  bool have_rho = false;
  std::vector<H> rr2(2 * nr), rho_next(nr);
  for (int64_t it = 1; it <= cfg.max_iters; ++it) {
    if (trace)
      std::fprintf(stderr, "[lrs] bicgstab it %lld host %.3f ms\n", (long long)it,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                             t_start).count());
    std::vector<bool> act(nr);
    for (int j = 0; j < nr; ++j) act[j] = !conv[j] && !brk[j];
    if (!any(act)) break;
    if (have_rho) rho = rho_next;
    else w.dots(rhat, 0, 1, r, rho.data());
    have_rho = false;
    for (int j = 0; j < nr; ++j)
      if (act[j] && std::abs(rho[j]) < cfg.breakdown_eps) {
        brk[j] = true;
        act[j] = false;
      }
    if (!any(act)) break;
    if (it == 1) {
      w.axpby(5, none, none, cs_mask(act), nullptr, r, nullptr, p);
    } else {
      std::vector<H> beta(nr, H(0.0));
      for (int j = 0; j < nr; ++j) beta[j] = (rho[j] / rho_prev[j]) * (alpha[j] / omega[j]);
      w.axpby(0, cs_fill<S>(beta), cs_fill<S>(omega), cs_mask(act), p, r, v, nullptr);
    }
    w.M(p, phat);
    w.Aop(phat, v);
    w.dots(rhat, 0, 1, v, rv.data());
    for (int j = 0; j < nr; ++j)
      if (act[j]) alpha[j] = rho[j] / (rv[j] != H(0.0) ? rv[j] : H(1.0));
    w.axpby(1, cs_fill<S>(alpha), none, cs_mask(act), nullptr, r, v, s);
    w.norms(s, tmpv.data());
    std::vector<bool> half(nr, false);
    for (int j = 0; j < nr; ++j) half[j] = act[j] && tmpv[j] / bns[j] <= cfg.tol;
    std::vector<bool> hist_cols = act;
    if (any(half)) {
      w.axpby(3, cs_fill<S>(alpha), none, cs_mask(half), x, phat, nullptr, tmp);
      // true residual of the candidate (columns outside `half` are stale and unused)
      w.resid(b, tmp, t);
      w.norms(t, tmpv2.data());
      std::vector<bool> ok(nr, false);
      for (int j = 0; j < nr; ++j) ok[j] = half[j] && tmpv2[j] / bns[j] <= cfg.tol;
      if (any(ok)) {
        w.axpby(5, none, none, cs_mask(ok), nullptr, tmp, nullptr, x);
        for (int j = 0; j < nr; ++j)
          if (ok[j]) {
            conv[j] = true;
            iters[j] = (double)it - 0.5;
            act[j] = false;
          }
      }
    }
    mx = 0;
    for (int j = 0; j < nr; ++j)
      if (hist_cols[j]) mx = std::max(mx, tmpv[j] / bns[j]);
    w.push(mx);
    if (!any(act)) break;
    w.M(s, shat);
    std::vector<H> st(2 * nr);
    w.Aop_dots2(shat, t, s, st.data());  // t = A shat, [s^H t, t^H t] (t follows s in buf)
    for (int j = 0; j < nr; ++j) {
      const H tt = st[nr + j], ts = hconj(st[j]);
      if (act[j]) omega[j] = ts / (tt != H(0.0) ? tt : H(1.0));
    }
    for (int j = 0; j < nr; ++j)
      if (act[j] && std::abs(omega[j]) < cfg.breakdown_eps) {
        brk[j] = true;
        act[j] = false;
      }
    w.axpby(2, cs_fill<S>(alpha), cs_fill<S>(omega), cs_mask(act), x, phat, shat, nullptr);
    w.axpby(1, cs_fill<S>(omega), none, cs_mask(act), nullptr, s, t, r);
    w.dots(r, (int64_t)blk, 2, r, rr2.data());  // [r^H r, rhat^H r] (rhat follows r)
    for (int j = 0; j < nr; ++j) {
      tmpv[j] = std::sqrt(hreal(rr2[j]));
      rho_next[j] = rr2[nr + j];
    }
    have_rho = true;
    std::vector<bool> full(nr, false);
    for (int j = 0; j < nr; ++j) full[j] = act[j] && tmpv[j] / bns[j] <= cfg.tol;
    if (any(full)) {
      w.resid(b, x, tmp);
      w.norms(tmp, tmpv2.data());
      for (int j = 0; j < nr; ++j)
        if (full[j] && tmpv2[j] / bns[j] <= cfg.tol) {
          conv[j] = true;
          iters[j] = (double)it;
        }
    }
    mx = 0;
    for (int j = 0; j < nr; ++j)
      if (act[j]) mx = std::max(mx, tmpv[j] / bns[j]);
    w.push(mx);
    for (int j = 0; j < nr; ++j) {
      if (act[j]) rho_prev[j] = rho[j];
      if (act[j] && !conv[j]) iters[j] = (double)it;
    }
  }
}

// Preconditioned CG, mirroring the checker's cg: iterations in
// BiCGStab half-iteration units (0.5 per CG step), true residual at claimed convergence.
template <class S>
void run_cg(Work<S>& w, const S* b, S* x, const lrs_iter_cfg& cfg, bool has_x0,
            std::vector<double>& iters, std::vector<bool>& conv, std::vector<bool>& brk) {
  using H = HT<S>;
  const int nr = w.nr;
  const int64_t n = w.n;
  const size_t blk = (size_t)n * nr;
  DevBuf<S> buf;
  buf.alloc(blk * 5);
  S* r = buf.get();
  S* z = r + blk;
  S* p = z + blk;
  S* q = p + blk;
  S* tmp = q + blk;
  const ColScalT<S> none{};
  std::vector<double> bn(nr), bns(nr), rres(nr), tr(nr);
  w.norms(b, bn.data());
  for (int j = 0; j < nr; ++j) bns[j] = bn[j] > 0 ? bn[j] : 1.0;
  if (has_x0) {
    w.resid(b, x, r);
  } else {
    w.zero(x);
    w.copy(r, b);
  }
  w.norms(r, rres.data());
  conv.assign(nr, false);
  brk.assign(nr, false);
  iters.assign(nr, 0.0);
  double mx = 0;
  for (int j = 0; j < nr; ++j) {
    conv[j] = rres[j] / bns[j] <= cfg.tol || bn[j] == 0.0;
    mx = std::max(mx, rres[j] / bns[j]);
  }
  w.push(mx);
  w.M(r, z);
  w.copy(p, z);
  std::vector<H> rz(nr), pq(nr), rzn(nr);
  w.dots(r, 0, 1, z, rz.data());
  for (int64_t it = 1; it <= cfg.max_iters; ++it) {
    std::vector<bool> act(nr);
    for (int j = 0; j < nr; ++j) act[j] = !conv[j] && !brk[j];
    if (!any(act)) break;
    for (int j = 0; j < nr; ++j)
      if (act[j] && std::abs(rz[j]) < cfg.breakdown_eps) {
        brk[j] = true;
        act[j] = false;
      }
    if (!any(act)) break;
    w.Aop(p, q);
    w.dots(p, 0, 1, q, pq.data());
    for (int j = 0; j < nr; ++j)
      if (act[j] && std::abs(pq[j]) < cfg.breakdown_eps) {
        brk[j] = true;
        act[j] = false;
      }
    if (!any(act)) break;
    std::vector<H> alpha(nr, H(0.0));
    for (int j = 0; j < nr; ++j)
      if (act[j]) alpha[j] = rz[j] / (pq[j] != H(0.0) ? pq[j] : H(1.0));
    w.axpby(2, cs_fill<S>(alpha), none, cs_mask(act), x, p, p, nullptr);  // x += alpha p
    w.axpby(1, cs_fill<S>(alpha), none, cs_mask(act), nullptr, r, q, r);  // r -= alpha q
    w.norms(r, rres.data());
    std::vector<bool> full(nr, false);
    for (int j = 0; j < nr; ++j) full[j] = act[j] && rres[j] / bns[j] <= cfg.tol;
    if (any(full)) {
      w.resid(b, x, tmp);
      w.norms(tmp, tr.data());
      for (int j = 0; j < nr; ++j)
        if (full[j] && tr[j] / bns[j] <= cfg.tol) {
          conv[j] = true;
          iters[j] = 0.5 * (double)it;
        }
    }
    mx = 0;
    for (int j = 0; j < nr; ++j)
      if (act[j]) mx = std::max(mx, rres[j] / bns[j]);
    w.push(mx);
    for (int j = 0; j < nr; ++j) {
      act[j] = act[j] && !conv[j];
      if (act[j]) iters[j] = 0.5 * (double)it;
    }
    if (!any(act)) break;
    w.M(r, z);
    w.dots(r, 0, 1, z, rzn.data());
    std::vector<H> beta(nr, H(0.0));
    for (int j = 0; j < nr; ++j)
      if (act[j]) beta[j] = rzn[j] / (rz[j] != H(0.0) ? rz[j] : H(1.0));
    w.axpby(0, cs_fill<S>(beta), none, cs_mask(act), p, z, p, nullptr);  // p = z + beta p
    for (int j = 0; j < nr; ++j)
      if (act[j]) rz[j] = rzn[j];
  }
}

// Givens rotation zeroing b against a: c real, c a + s b = d, -conj(s) a + c b = 0.
template <class H>
void givens(H a, H b, double* c, H* s, H* d) {
  if (b == H(0.0)) {
    *c = 1.0;
    *s = H(0.0);
    *d = a;
    return;
  }
  if (a == H(0.0)) {
    *c = 0.0;
    *s = hconj(b) / std::abs(b);
    *d = H(std::abs(b));
    return;
  }
  const double na = std::abs(a), nb = std::abs(b);
  const double dd = std::hypot(na, nb);
  const H sa = a / na;
  *c = na / dd;
  *s = sa * hconj(b) / dd;
  *d = sa * dd;
}

template <class S>
void run_gmres(Work<S>& w, const S* b, S* x, const lrs_iter_cfg& cfg, bool has_x0,
               std::vector<double>& iters_out, std::vector<bool>& conv) {
  using H = HT<S>;
  const int nr = w.nr;
  const int64_t n = w.n;
  const int m = std::max(1, (int)cfg.restart);
  if (m + 1 > 64) throw LrsError(LRS_ERR_PARAMETER, "GMRES restart must be <= 63");
  Ctx* c = w.c();
  const size_t blk = (size_t)n * nr;
  DevBuf<S> buf;
  buf.alloc(blk * (2 * (size_t)m + 3));
  S* V = buf.get();               // (m+1) blocks
  S* Z = V + blk * (m + 1);       // m blocks
  S* wv = Z + blk * m;
  S* r = wv + blk;
  DevBuf<S> ydev;
  ydev.alloc((size_t)(m + 1) * MAX_RHS);
  const ColScalT<S> none{};
  std::vector<double> bn(nr), bns(nr), beta(nr);
  w.norms(b, bn.data());
  for (int j = 0; j < nr; ++j) bns[j] = bn[j] > 0 ? bn[j] : 1.0;
  if (has_x0) {
    w.resid(b, x, r);
  } else {
    w.zero(x);
    w.copy(r, b);
  }
  w.norms(r, beta.data());
  conv.assign(nr, false);
  std::vector<int64_t> iters(nr, 0);
  double mx = 0;
  for (int j = 0; j < nr; ++j) {
    conv[j] = beta[j] / bns[j] <= cfg.tol || bn[j] == 0.0;
    mx = std::max(mx, beta[j] / bns[j]);
  }
  w.push(mx);
  const std::vector<bool> all(nr, true);
  std::vector<H> h((m + 1) * nr), h2((m + 1) * nr);
  std::vector<double> hn(nr);
  while (true) {
    std::vector<bool> act(nr);
    for (int j = 0; j < nr; ++j) act[j] = !conv[j] && iters[j] < cfg.max_iters;
    if (!any(act)) break;
    std::vector<H> inv(nr);
    for (int j = 0; j < nr; ++j) inv[j] = H(1.0 / (beta[j] > 0 ? beta[j] : 1.0));
    w.axpby(4, cs_fill<S>(inv), none, cs_mask(all), nullptr, r, nullptr, V);
    // per column Hessenberg (after rotations) R[row + col*(m+1)], g, rotations
    std::vector<std::vector<H>> R(nr, std::vector<H>((size_t)(m + 1) * m, H(0.0)));
    std::vector<std::vector<H>> g(nr, std::vector<H>(m + 1, H(0.0)));
    std::vector<std::vector<double>> csv(nr, std::vector<double>(m, 0.0));
    std::vector<std::vector<H>> snv(nr, std::vector<H>(m, H(0.0)));
    for (int j = 0; j < nr; ++j) g[j][0] = H(beta[j]);
    std::vector<bool> inner = act;
    std::vector<int> steps(nr, 0);
    for (int jj = 0; jj < m; ++jj) {
      if (!any(inner)) break;
      S* Vj = V + blk * jj;
      S* Zj = Z + blk * jj;
      w.M(Vj, Zj);
      w.Aop(Zj, wv);
      // CGS2 (the projections stay on the device in dotout and feed the update directly;
      // the host reads h, h2 and the norm after one synchronization)
      w.dots_enqueue(V, (int64_t)blk, jj + 1, wv, 0);
      launch_multi_axpy_t<S>(c, w.nl, nr, V + w.lo, n, (int64_t)blk, jj + 1, w.dotout(), -1.0,
                             wv + w.lo, n);
      w.dots_enqueue(V, (int64_t)blk, jj + 1, wv, 1);
      launch_multi_axpy_t<S>(c, w.nl, nr, V + w.lo, n, (int64_t)blk, jj + 1, w.dotout(), -1.0,
                             wv + w.lo, n);
      w.dots_enqueue(wv, 0, 1, wv, 2);
      w.dots_wait();
      w.dots_read(jj + 1, 0, h.data());
      w.dots_read(jj + 1, 1, h2.data());
      {
        std::vector<H> nn(nr);
        w.dots_read(1, 2, nn.data());
        for (int j = 0; j < nr; ++j) hn[j] = std::sqrt(hreal(nn[j]));
      }
      for (int q = 0; q < (jj + 1) * nr; ++q) h[q] += h2[q];
      std::vector<H> invn(nr);
      for (int j = 0; j < nr; ++j) invn[j] = H(1.0 / (hn[j] > 0 ? hn[j] : 1.0));
      w.axpby(4, cs_fill<S>(invn), none, cs_mask(all), nullptr, wv, nullptr, V + blk * (jj + 1));
      mx = 0;
      for (int j = 0; j < nr; ++j) {
        if (!inner[j]) continue;
        std::vector<H> col(m + 1, H(0.0));
        for (int q = 0; q <= jj; ++q) col[q] = h[q * nr + j];
        col[jj + 1] = H(hn[j]);
        for (int q = 0; q < jj; ++q) {
          const H t = csv[j][q] * col[q] + snv[j][q] * col[q + 1];
          col[q + 1] = -hconj(snv[j][q]) * col[q] + csv[j][q] * col[q + 1];
          col[q] = t;
        }
        double cc;
        H ss, d;
        givens<H>(col[jj], col[jj + 1], &cc, &ss, &d);
        csv[j][jj] = cc;
        snv[j][jj] = ss;
        col[jj] = d;
        col[jj + 1] = H(0.0);
        g[j][jj + 1] = -hconj(ss) * g[j][jj];
        g[j][jj] = cc * g[j][jj];
        for (int q = 0; q <= jj; ++q) R[j][q + (size_t)jj * (m + 1)] = col[q];
        steps[j]++;
        iters[j]++;
      }
      for (int j = 0; j < nr; ++j) {
        if (!inner[j]) continue;
        const double est = std::abs(g[j][jj + 1]) / bns[j];
        mx = std::max(mx, est);
        if (!(est > cfg.tol) || iters[j] >= cfg.max_iters) inner[j] = false;
      }
      w.push(mx);
    }
    // x += Z y per active column
    int kmax = 0;
    for (int j = 0; j < nr; ++j)
      if (act[j]) kmax = std::max(kmax, steps[j]);
    if (kmax > 0) {
      std::vector<H> y((size_t)kmax * nr, H(0.0));
      for (int j = 0; j < nr; ++j) {
        if (!act[j] || steps[j] == 0) continue;
        const int kk = steps[j];
        std::vector<H> yy(kk);
        for (int q = kk - 1; q >= 0; --q) {
          H s = g[j][q];
          for (int e = q + 1; e < kk; ++e) s -= R[j][q + (size_t)e * (m + 1)] * yy[e];
          yy[q] = s / R[j][q + (size_t)q * (m + 1)];
        }
        for (int q = 0; q < kk; ++q) y[(size_t)q * nr + j] = yy[q];
      }
      c->stage_h2d(ydev.get(), y.data(), sizeof(H) * y.size());
      launch_multi_axpy_t<S>(c, w.nl, nr, Z + w.lo, n, (int64_t)blk, kmax, ydev.get(), 1.0,
                             x + w.lo, n);
      LRS_CUDA(cudaStreamSynchronize(c->stream));
    }
    w.resid(b, x, r);
    w.norms(r, hn.data());
    for (int j = 0; j < nr; ++j)
      if (act[j]) {
        beta[j] = hn[j];
        if (beta[j] / bns[j] <= cfg.tol) conv[j] = true;
      }
  }
  iters_out.assign(nr, 0.0);
  for (int j = 0; j < nr; ++j) iters_out[j] = (double)iters[j];
}

// ------------------------------------------------------------------------------------
// The reduced system of LR-SPIKE-I / OTF in the compact layout (reduced.cu)
// ------------------------------------------------------------------------------------
template <class S>
const IfaceApplyJobT<S>* red_jobs(Fact* f) {
  return reinterpret_cast<const IfaceApplyJobT<S>*>(f->iface_jobs_red.get());
}

// the two compressed messages of every local-side interface of a compact vector (C1)
template <class S>
void reduced_messages(Fact* f, const S* xr, int nr) {
  launch_iface_messages_t<S>(f->ctx, red_jobs<S>(f), f->ni, f->r, f->k, xr, f->ldr, nr,
                             sp<S>(f->iface_work));
  exchange_msgs<S>(f, nr);
}

// matvec_lowrank: y = x + W~ x_{i-1,b} + T~ x_{i+1,t}
template <class S>
void matvec_lowrank_t(Fact* f, const S* x, S* y, int nr) {
  reduced_messages(f, x, nr);
  launch_iface_scale_t<S>(f->ctx, red_jobs<S>(f), f->ni, f->r, nr);
  launch_tips_lowrank_t<S>(f->ctx, f->geom(), f->n, f->k, x, y, f->ldr, nr, sp<S>(f->uT),
                           sp<S>(f->uW), f->r, sp<S>(f->scT), sp<S>(f->scW), 0, 1.0);
  ledger_add(f, LRS_STAGE_REDUCED_MATVEC, 2, (int64_t)f->r * nr);
}

// apply_truncated_precond on a compact vector
template <class S>
void trunc_precond_t(Fact* f, const S* g, S* x, int nr) {
  reduced_messages(f, g, nr);
  launch_iface_solve_t<S>(f->ctx, red_jobs<S>(f), f->ni, f->r, nr);
  launch_tips_lowrank_t<S>(f->ctx, f->geom(), f->n, f->k, g, x, f->ldr, nr, sp<S>(f->uT),
                           sp<S>(f->uW), f->r, sp<S>(f->scT), sp<S>(f->scW), 1, -1.0);
  ledger_add(f, LRS_STAGE_PRECOND_APPLY, 2, (int64_t)f->r * nr);
}

// z (n-layout, zeroed local rows) = A_i^-1 (pad_top(C_i x_{i-1,b}) + pad_bottom(B_i x_{i+1,t}))
// for the local partitions, x compact (exact spikes applied on the fly);
// the neighbour tips of the cross-GPU interfaces arrive by a neighbour exchange.
template <class S>
void coupled_solve_t(Fact* f, S* xr, S* z, int nr) {
  Ctx* c = f->ctx;
  const int64_t k = f->k, n = f->n, ldr = f->ldr, k2 = 2 * k;
  if (f->dist) {  // x_{p0-1,b} from the left GPU, x_{p0+P,t} from the right GPU
    const int64_t cnt = k * nr;
    S* s_next = sp<S>(f->xch);
    S* s_prev = s_next + cnt;
    S* r_prev = s_prev + cnt;
    S* r_next = r_prev + cnt;
    copy_block(c, s_next, k, xr + k2 * (f->p0 + f->P - 1) + k, ldr, k, nr);
    copy_block(c, s_prev, k, xr + k2 * f->p0, ldr, k, nr);
    neighbor_exchange(f, s_next, r_prev, s_prev, r_next, cnt * SW<S>);
    if (f->p0 > 0) copy_block(c, xr + k2 * (f->p0 - 1) + k, ldr, r_prev, k, k, nr);
    if (f->p0 + f->P < f->Pg) copy_block(c, xr + k2 * (f->p0 + f->P), ldr, r_next, k, k, nr);
  }
  for (int j = 0; j < nr; ++j)
    LRS_CUDA(cudaMemsetAsync(z + f->row_lo + (int64_t)j * n, 0,
                             sizeof(S) * (f->row_hi - f->row_lo), c->stream));
  std::vector<CoupleJobT<S>> wj, tj;
  for (int i = f->p0; i < f->p0 + f->P; ++i) {
    const int64_t o = f->goff[i], ni = f->goff[i + 1] - f->goff[i];
    if (i > 0) {  // C_i x_{i-1,b} into the top k rows
      CoupleJobT<S> j{};
      j.r0 = o;
      j.c0 = o - k;
      j.b = k;
      j.dst0 = o;
      j.X = xr + k2 * (i - 1) + k;
      j.ldx = ldr;
      j.out = z;
      j.ldo = n;
      j.ncols = nr;
      wj.push_back(j);
    }
    if (i < f->Pg - 1) {  // B_i x_{i+1,t} into the bottom k rows
      CoupleJobT<S> j{};
      j.r0 = o + ni - k;
      j.c0 = f->goff[i + 1];
      j.b = k;
      j.dst0 = o + ni - k;
      j.X = xr + k2 * (i + 1);
      j.ldx = ldr;
      j.out = z;
      j.ldo = n;
      j.ncols = nr;
      tj.push_back(j);
    }
  }
  DevBuf<CoupleJobT<S>> dw, dt;
  upload(c, dw, wj);
  upload(c, dt, tj);
  launch_coupling_t<S>(c, f->mat, false, dw.get(), (int)wj.size(), k, nr, true);
  launch_coupling_t<S>(c, f->mat, false, dt.get(), (int)tj.size(), k, nr, true);
  dstage_t(f, z, n, nr, false, -1);
}

// matvec_otf: y = x + tips(z), z from coupled_solve_t
template <class S>
void matvec_otf_t(Fact* f, S* x, S* y, S* z, int nr) {
  coupled_solve_t(f, x, z, nr);
  launch_tips_gather_t<S>(f->ctx, f->geom(), f->k, z, f->n, x, y, f->ldr, nr);
  ledger_add(f, LRS_STAGE_REDUCED_MATVEC, 2, f->k * nr);
}

template <class S>
void reduced_work(Work<S>& w, Fact* f, int nr, lrs_report* rep) {
  w.f = f;
  w.n = f->ldr;
  w.lo = 2 * f->k * f->p0;
  w.nl = 2 * f->k * f->P;
  w.ch = f->rchunks();
  w.nr = nr;
  w.rep = rep;
  w.init();
}

template <class S>
ColScalT<S> cs_const(int nr, double v) {
  ColScalT<S> s{};
  for (int j = 0; j < nr && j < MAX_RHS; ++j) s.v[j] = s_real<S>(v);
  return s;
}

// apply_precond_I: D-stage; inner BiCGStab on the low-rank reduced
// system (matvec_lowrank, preconditioned by apply_truncated_precond) on the column-
// normalised tips; low-rank recovery.  Inner non-convergence -> LRS_ERR_PRECOND_FAILURE.
template <class S>
void apply_precond_I_t(Fact* f, const S* in, int64_t ldi, S* out, int64_t ldo, int nrhs) {
  Ctx* c = f->ctx;
  const int64_t nl = f->row_hi - f->row_lo;
  if (out != in) copy_block(c, out + f->row_lo, ldo, in + f->row_lo, ldi, nl, nrhs);
  dstage_t(f, out, ldo, nrhs, false, -1);
  if (!(f->r > 0 && f->Pg > 1)) return;
  for (int c0 = 0; c0 < nrhs; c0 += MAX_RHS) {
    const int nr = std::min(MAX_RHS, nrhs - c0);
    S* y = out + (int64_t)c0 * ldo;
    DevBuf<S> rb;
    rb.alloc((size_t)f->ldr * nr * 2);
    S* g = rb.get();
    S* xr = g + (size_t)f->ldr * nr;
    launch_tips_gather_t<S>(c, f->geom(), f->k, y, ldo, nullptr, g, f->ldr, nr);
    lrs_report irep{};
    Work<S> wi;
    reduced_work(wi, f, nr, &irep);
    wi.Af = [&](S* a, S* o) { matvec_lowrank_t(f, a, o, nr); };
    wi.Mf = [&](const S* a, S* o) { trunc_precond_t(f, a, o, nr); };
    wi.Rf = [&](const S* b, S* xx, S* o) {
      matvec_lowrank_t(f, xx, o, nr);
      wi.axpby(1, cs_const<S>(nr, 1.0), ColScalT<S>{}, cs_const<double>(nr, 1.0), nullptr, b, o, o);
    };
    std::vector<double> gn(nr);
    wi.norms(g, gn.data());
    ColScalT<S> inv{}, scl{};
    for (int j = 0; j < nr; ++j) {
      const double gs = gn[j] > 0 ? gn[j] : 1.0;
      inv.v[j] = s_real<S>(1.0 / gs);
      scl.v[j] = s_real<S>(gs);
    }
    const ColScal all = cs_const<double>(nr, 1.0);
    wi.axpby(4, inv, ColScalT<S>{}, all, nullptr, g, nullptr, g);
    lrs_iter_cfg icfg{};
    icfg.method = LRS_BICGSTAB;
    icfg.tol = f->inner_tol;
    icfg.max_iters = f->inner_max_iters;
    icfg.breakdown_eps = 1e-30;
    std::vector<double> its;
    std::vector<bool> conv, brk;
    run_bicgstab(wi, g, xr, icfg, false, its, conv, brk);
    bool ok = true;
    double itmax = 0.0;
    for (int j = 0; j < nr; ++j) {
      ok = ok && conv[j] && !brk[j];
      itmax = std::max(itmax, its[j]);
    }
    if (!ok)
      throw LrsError(LRS_ERR_PRECOND_FAILURE,
                     "LR-SPIKE-I inner reduced solve did not converge (tol " +
                         std::to_string(f->inner_tol) + ", " + std::to_string(icfg.max_iters) +
                         " iterations)");
    f->inner_iterations += itmax;
    f->inner_solves += 1;
    wi.axpby(4, scl, ColScalT<S>{}, all, nullptr, xr, nullptr, xr);
    // low-rank recovery with the reduced solution's compressed messages
    reduced_messages(f, xr, nr);
    launch_iface_scale_t<S>(c, red_jobs<S>(f), f->ni, f->r, nr);
    launch_recovery_t<S>(c, f->geom(), f->n, f->row_lo, f->row_hi, y, ldo, y, ldo, nr,
                         sp<S>(f->uT), sp<S>(f->uW), f->r, sp<S>(f->scT), sp<S>(f->scW));
    ledger_add(f, LRS_STAGE_RECOVERY, 2, (int64_t)f->r * nr);
  }
}

// mode APPLY_VARIANT: the factorization's own preconditioner (I for LR-SPIKE-I, Block
// Jacobi for BJ, T otherwise); APPLY_BJ: the D-stage only; APPLY_T: apply_precond_T
template <class S>
void apply_variant_t(Fact* f, const S* in, int64_t ldi, S* out, int64_t ldo, int nrhs, int mode) {
  if (mode == APPLY_VARIANT && f->variant == LRS_VARIANT_I)
    apply_precond_I_t(f, in, ldi, out, ldo, nrhs);
  else
    apply_precond_t(f, in, ldi, out, ldo, nrhs,
                    mode == APPLY_BJ || (mode == APPLY_VARIANT && f->variant == LRS_VARIANT_BJ));
}

// solve_otf for one column batch: D-stage once; BiCGStab on the true
// reduced system (matvec_otf) preconditioned by apply_truncated_precond to otf_tol;
// exact recovery x = y - z(x_r); full residual against the outer tol, escalating the
// reduced tolerance /100 (warm restart) at most otf_escalations times.
template <class S>
void run_otf(Work<S>& w, Fact* f, const S* b, S* x, const lrs_iter_cfg& cfg,
             std::vector<double>& iters, std::vector<bool>& conv, std::vector<bool>& brk) {
  Ctx* c = f->ctx;
  const int nr = w.nr;
  const int64_t n = f->n;
  const size_t blk = (size_t)n * nr;
  DevBuf<S> buf;
  buf.alloc(blk * 3);
  S* y = buf.get();
  S* z = y + blk;
  S* t = z + blk;
  std::vector<double> bn(nr), res(nr);
  w.norms(b, bn.data());
  w.copy(y, b);
  dstage_t(f, y, n, nr, false, -1);
  w.rep->precond_applications++;
  iters.assign(nr, 0.0);
  conv.assign(nr, false);
  brk.assign(nr, false);
  auto check = [&]() {
    w.resid(b, x, t);
    w.norms(t, res.data());
    bool all = true;
    double mx = 0.0;
    for (int j = 0; j < nr; ++j) {
      const double rr = res[j] / (bn[j] > 0 ? bn[j] : 1.0);
      mx = std::max(mx, rr);
      all = all && rr <= cfg.tol;
    }
    return std::make_pair(all, mx);
  };
  if (!f->coupled) {  // S_r = I: x = D^-1 f, zero reduced iterations
    w.copy(x, y);
    const auto ck = check();
    conv.assign(nr, ck.first);
    return;
  }
  DevBuf<S> rb;
  rb.alloc((size_t)f->ldr * nr * 2);
  S* g = rb.get();
  S* xr = g + (size_t)f->ldr * nr;
  launch_tips_gather_t<S>(c, f->geom(), f->k, y, n, nullptr, g, f->ldr, nr);
  lrs_report rrep{};
  Work<S> wr;
  reduced_work(wr, f, nr, &rrep);
  wr.Af = [&](S* a, S* o) { matvec_otf_t(f, a, o, z, nr); };
  if (f->r > 0) wr.Mf = [&](const S* a, S* o) { trunc_precond_t(f, a, o, nr); };
  else wr.Mf = [&](const S* a, S* o) { copy_block(c, o + wr.lo, wr.n, a + wr.lo, wr.n, wr.nl, nr); };
  wr.Rf = [&](const S* bb, S* xx, S* o) {
    matvec_otf_t(f, xx, o, z, nr);
    wr.axpby(1, cs_const<S>(nr, 1.0), ColScalT<S>{}, cs_const<double>(nr, 1.0), nullptr, bb, o, o);
  };
  double tol = f->otf_tol, total = 0.0;
  bool warm = false;
  const ColScal all = cs_const<double>(nr, 1.0);
  for (int esc = 0; esc <= f->otf_escalations; ++esc) {
    lrs_iter_cfg rcfg{};
    rcfg.method = LRS_BICGSTAB;
    rcfg.tol = tol;
    rcfg.max_iters = f->otf_max_iters;
    rcfg.breakdown_eps = cfg.breakdown_eps;
    std::vector<double> its;
    std::vector<bool> rc, rbrk;
    run_bicgstab(wr, g, xr, rcfg, warm, its, rc, rbrk);
    double itmax = 0.0;
    for (int j = 0; j < nr; ++j) {
      itmax = std::max(itmax, its[j]);
      if (rbrk[j]) brk[j] = true;
    }
    total += itmax;
    w.hist.insert(w.hist.end(), wr.hist.begin(), wr.hist.end());
    wr.hist.clear();
    if (std::any_of(brk.begin(), brk.end(), [](bool v) { return v; })) break;
    // exact recovery x = y - z(x_r)
    coupled_solve_t(f, xr, z, nr);
    ledger_add(f, LRS_STAGE_RECOVERY, 2, f->k * nr);
    w.axpby(1, cs_const<S>(nr, 1.0), ColScalT<S>{}, all, nullptr, y, z, x);
    const auto ck = check();
    if (ck.first) {
      conv.assign(nr, true);
      break;
    }
    tol /= 100.0;
    warm = true;
  }
  w.rep->matvecs += rrep.matvecs;
  for (int j = 0; j < nr; ++j) iters[j] = total;
}

template <class S>
void solve_t(Fact* f, Mat* a, const S* b, int64_t ldb, S* x, int64_t ldx, int nrhs,
             const lrs_iter_cfg& cfg, lrs_report* rep) {
  Ctx* c = f->ctx;
  const int64_t m0[3] = {f->ledger_msgs[0], f->ledger_msgs[1], f->ledger_msgs[2]};
  const int64_t s0[3] = {f->ledger_sc[0], f->ledger_sc[1], f->ledger_sc[2]};
  lrs_report& R = *rep;
  double* hist_buf = R.history;
  const int64_t cap = R.history_cap;
  std::memset(&R, 0, sizeof(R));
  R.history = hist_buf;
  R.history_cap = cap;
  R.seed = f->seed;
  R.converged = 1;
  const int64_t calls0 = f->comm_calls, csync0 = f->comm_syncs, ssync0 = f->scalar_syncs;
  const double inner0 = f->inner_iterations;
  const int64_t solves0 = f->inner_solves;
  LRS_CUDA(cudaEventRecord(c->ev0, c->stream));
  const int64_t n = f->n, lo = f->row_lo, nl = f->row_hi - f->row_lo;
  bool any_brk = false;
  double worst = 0.0;
  std::vector<double> hist_all;
  for (int c0 = 0; c0 < nrhs; c0 += MAX_RHS) {
    const int nr = std::min(MAX_RHS, nrhs - c0);
    Work<S> w;
    w.f = f;
    w.n = n;
    w.lo = lo;
    w.nl = nl;
    w.ch = f->chunks();
    w.nr = nr;
    w.rep = &R;
    w.init();
    w.Mf = [&](const S* in, S* out) { apply_variant_t(f, in, n, out, n, nr, APPLY_VARIANT); };
    w.Af = [&](S* in, S* out) {
      halo_exchange(f, in, n, nr);
      spmv_s<S>(c, a, in, n, out, n, nr, 0, nullptr, 0, lo, lo + nl);
    };
    w.Rf = [&](const S* bv, S* xv, S* out) {
      halo_exchange(f, xv, n, nr);
      spmv_s<S>(c, a, xv, n, out, n, nr, 2, bv, n, lo, lo + nl);
    };
    if (!spmv_dot_unfused())
      w.AfD = [&](S* in, S* out, const S* X) {
        halo_exchange(f, in, n, nr);
        launch_spmv_dot2_t<S>(c, a, w.ch, in, n, out, n, nr, X, n, sp<S>(f->partial));
      };
    // full-length device copies (ld = n) of this column batch; local rows only
    DevBuf<S> bb, xx;
    bb.alloc((size_t)n * nr);
    xx.alloc((size_t)n * nr);
    copy_block(c, bb.get() + lo, n, b + (int64_t)c0 * ldb + lo, ldb, nl, nr);
    const bool has_x0 = cfg.x0 != nullptr;
    if (has_x0)
      copy_block(c, xx.get() + lo, n, static_cast<const S*>(cfg.x0) + (int64_t)c0 * ldx + lo, ldx,
                 nl, nr);
    std::vector<double> iters;
    std::vector<bool> conv, brk;
    if (f->variant == LRS_VARIANT_OTF) {
      run_otf(w, f, bb.get(), xx.get(), cfg, iters, conv, brk);
    } else if (cfg.method == LRS_BICGSTAB) {
      run_bicgstab(w, bb.get(), xx.get(), cfg, has_x0, iters, conv, brk);
    } else if (cfg.method == LRS_GMRES) {
      run_gmres(w, bb.get(), xx.get(), cfg, has_x0, iters, conv);
      brk.assign(nr, false);
    } else if (cfg.method == LRS_CG) {
      run_cg(w, bb.get(), xx.get(), cfg, has_x0, iters, conv, brk);
    } else {
      throw LrsError(LRS_ERR_PARAMETER, "unknown Krylov method");
    }
    for (int j = 0; j < nr; ++j) {
      R.iterations = std::max(R.iterations, iters[j]);
      if (!conv[j]) R.converged = 0;
      if (brk[j]) any_brk = true;
    }
    // final true residual (not counted as a solver matvec)
    {
      std::vector<double> bn(nr), rn(nr);
      w.norms(bb.get(), bn.data());
      DevBuf<S> tmp;
      tmp.alloc((size_t)n * nr);
      halo_exchange(f, xx.get(), n, nr);
      spmv_s<S>(c, a, xx.get(), n, tmp.get(), n, nr, 2, bb.get(), n, lo, lo + nl);
      w.norms(tmp.get(), rn.data());
      for (int j = 0; j < nr; ++j) worst = std::max(worst, rn[j] / (bn[j] > 0 ? bn[j] : 1.0));
    }
    copy_block(c, x + (int64_t)c0 * ldx + lo, ldx, xx.get() + lo, n, nl, nr);
    hist_all.insert(hist_all.end(), w.hist.begin(), w.hist.end());
  }
  LRS_CUDA(cudaEventRecord(c->ev1, c->stream));
  LRS_CUDA(cudaEventSynchronize(c->ev1));
  R.t_solve = elapsed_ms(c->ev0, c->ev1) * 1e-3;
  R.residual_final = worst;
  R.comm_calls = f->comm_calls - calls0;
  R.comm_host_syncs = f->comm_syncs - csync0;
  R.scalar_syncs = f->scalar_syncs - ssync0;
  R.breakdown = any_brk ? 1 : 0;
  R.inner_iterations = f->inner_iterations - inner0;
  R.inner_solves = f->inner_solves - solves0;
  for (int s = 0; s < 3; ++s) {
    R.comm_messages[s] = f->ledger_msgs[s] - m0[s];
    R.comm_scalars[s] = f->ledger_sc[s] - s0[s];
  }
  R.history_total = (int64_t)hist_all.size();
  R.history_len = 0;
  if (R.history && R.history_cap > 0) {
    R.history_len = std::min<int64_t>(R.history_cap, (int64_t)hist_all.size());
    std::memcpy(R.history, hist_all.data(), sizeof(double) * R.history_len);
  }
  if (any_brk)
    throw LrsError(LRS_ERR_BREAKDOWN, cfg.method == LRS_CG
                                          ? "CG breakdown (|p^H A p| or |r^H z| below breakdown_eps)"
                                          : "BiCGStab stagnation detected (SF)");
}

}  // namespace

void solve(Fact* f, Mat* a, const void* b, int64_t ldb, void* x, int64_t ldx, int nrhs,
           const lrs_iter_cfg& cfg, lrs_report* rep) {
  if (a->n != f->n) throw LrsError(LRS_ERR_DIMENSION, "solve: matrix does not match factorization");
  if (a->scalar != f->scalar)
    throw LrsError(LRS_ERR_PARAMETER, "solve: matrix scalar type does not match factorization");
  if (cfg.tol <= 0 || cfg.max_iters < 1) throw LrsError(LRS_ERR_PARAMETER, "tol > 0 and max_iters >= 1");
  if (f->scalar == LRS_C128)
    solve_t(f, a, static_cast<const zc*>(b), ldb, static_cast<zc*>(x), ldx, nrhs, cfg, rep);
  else
    solve_t(f, a, static_cast<const double*>(b), ldb, static_cast<double*>(x), ldx, nrhs, cfg, rep);
}

// ------------------------------------------------------------------------------------
// Krylov drivers on caller-supplied operators (bicgstab / cg take
// abstract operator and preconditioner contracts; GMRES(m) likewise).  The space is one
// "partition" of n rows with the same deterministic chunked reductions.
// ------------------------------------------------------------------------------------
template <class S>
void krylov_ops_t(Ctx* c, int64_t n, const lrs_operator& A, const lrs_operator* M, const S* b,
                  int64_t ldb, S* x, int64_t ldx, int nrhs, const lrs_iter_cfg& cfg,
                  lrs_report* rep) {
  if (n < 1) throw LrsError(LRS_ERR_DIMENSION, "krylov: n >= 1 required");
  if (!A.apply) throw LrsError(LRS_ERR_PARAMETER, "krylov: apply_A callback required");
  if (cfg.tol <= 0 || cfg.max_iters < 1) throw LrsError(LRS_ERR_PARAMETER, "tol > 0 and max_iters >= 1");
  constexpr int w = SW<S>;
  Fact sp_;  // the reduction machinery of a one-partition space (no factors)
  Fact* f = &sp_;
  f->ctx = c;
  f->scalar = IsC<S>::value ? LRS_C128 : LRS_F64;
  f->sw = w;
  f->P = f->Pg = 1;
  f->n = n;
  f->row_lo = 0;
  f->row_hi = n;
  f->rank_pl.assign(1, 1);
  f->pl_max = 1;
  upload(c, f->d_rank_pl, f->rank_pl);
  const int64_t CH = KRYLOV_CHUNK;
  for (int64_t r0 = 0; r0 < n; r0 += CH) f->chunk_start.push_back(r0);
  f->part_first = {0, (int)f->chunk_start.size()};
  f->chunk_start.push_back(n);
  upload(c, f->d_chunks, f->chunk_start);
  upload(c, f->d_part_first, f->part_first);
  f->partial.alloc((f->chunk_start.size() - 1) * 64 * MAX_RHS * w);
  f->persum.alloc((size_t)64 * MAX_RHS * w);
  f->gather.alloc((size_t)64 * MAX_RHS * w);
  f->dotout.alloc((size_t)64 * MAX_RHS * w);
  lrs_report& R = *rep;
  double* hist_buf = R.history;
  const int64_t cap = R.history_cap;
  std::memset(&R, 0, sizeof(R));
  R.history = hist_buf;
  R.history_cap = cap;
  R.converged = 1;
  LRS_CUDA(cudaEventRecord(c->ev0, c->stream));
  bool any_brk = false;
  double worst = 0.0;
  std::vector<double> hist_all;
  auto call = [&](const lrs_operator& op, const S* in, S* out, int nr) {
    LRS_CUDA(cudaStreamSynchronize(c->stream));
    if (op.apply(op.user, in, out, n, nr) != 0)
      throw LrsError(LRS_ERR_PARAMETER, "krylov: operator callback failed");
  };
  for (int c0 = 0; c0 < nrhs; c0 += MAX_RHS) {
    const int nr = std::min(MAX_RHS, nrhs - c0);
    Work<S> wk;
    wk.f = f;
    wk.n = n;
    wk.lo = 0;
    wk.nl = n;
    wk.ch = f->chunks();
    wk.nr = nr;
    wk.rep = &R;
    wk.init();
    DevBuf<S> bb, xx, tmp;
    bb.alloc((size_t)n * nr);
    xx.alloc((size_t)n * nr);
    tmp.alloc((size_t)n * nr);
    copy_block(c, bb.get(), n, b + (int64_t)c0 * ldb, ldb, n, nr);
    const bool has_x0 = cfg.x0 != nullptr;
    if (has_x0)
      copy_block(c, xx.get(), n, static_cast<const S*>(cfg.x0) + (int64_t)c0 * ldx, ldx, n, nr);
    wk.Af = [&](S* in, S* out) { call(A, in, out, nr); };
    if (M && M->apply) wk.Mf = [&](const S* in, S* out) { call(*M, in, out, nr); };
    else wk.Mf = [&](const S* in, S* out) { copy_block(c, out, n, in, n, n, nr); };
    wk.Rf = [&](const S* bv, S* xv, S* out) {
      call(A, xv, out, nr);
      wk.axpby(1, cs_const<S>(nr, 1.0), ColScalT<S>{}, cs_const<double>(nr, 1.0), nullptr, bv, out,
               out);
    };
    std::vector<double> iters;
    std::vector<bool> conv, brk;
    if (cfg.method == LRS_BICGSTAB) {
      run_bicgstab(wk, bb.get(), xx.get(), cfg, has_x0, iters, conv, brk);
    } else if (cfg.method == LRS_GMRES) {
      run_gmres(wk, bb.get(), xx.get(), cfg, has_x0, iters, conv);
      brk.assign(nr, false);
    } else if (cfg.method == LRS_CG) {
      run_cg(wk, bb.get(), xx.get(), cfg, has_x0, iters, conv, brk);
    } else {
      throw LrsError(LRS_ERR_PARAMETER, "unknown Krylov method");
    }
    for (int j = 0; j < nr; ++j) {
      R.iterations = std::max(R.iterations, iters[j]);
      if (!conv[j]) R.converged = 0;
      if (brk[j]) any_brk = true;
    }
    std::vector<double> bn(nr), rn(nr);
    wk.norms(bb.get(), bn.data());
    wk.Rf(bb.get(), xx.get(), tmp.get());
    wk.norms(tmp.get(), rn.data());
    for (int j = 0; j < nr; ++j) worst = std::max(worst, rn[j] / (bn[j] > 0 ? bn[j] : 1.0));
    copy_block(c, x + (int64_t)c0 * ldx, ldx, xx.get(), n, n, nr);
    hist_all.insert(hist_all.end(), wk.hist.begin(), wk.hist.end());
  }
  LRS_CUDA(cudaEventRecord(c->ev1, c->stream));
  LRS_CUDA(cudaEventSynchronize(c->ev1));
  R.t_solve = elapsed_ms(c->ev0, c->ev1) * 1e-3;
  R.residual_final = worst;
  R.breakdown = any_brk ? 1 : 0;
  R.history_total = (int64_t)hist_all.size();
  if (R.history && R.history_cap > 0) {
    R.history_len = std::min<int64_t>(R.history_cap, (int64_t)hist_all.size());
    std::memcpy(R.history, hist_all.data(), sizeof(double) * R.history_len);
  }
  if (any_brk)
    throw LrsError(LRS_ERR_BREAKDOWN, cfg.method == LRS_CG ? "CG breakdown" : "BiCGStab stagnation detected (SF)");
}

void krylov_ops(Ctx* c, int64_t n, int32_t scalar, const lrs_operator& A, const lrs_operator* M,
                const void* b, int64_t ldb, void* x, int64_t ldx, int nrhs,
                const lrs_iter_cfg& cfg, lrs_report* rep) {
  if (scalar == LRS_C128)
    krylov_ops_t(c, n, A, M, static_cast<const zc*>(b), ldb, static_cast<zc*>(x), ldx, nrhs, cfg,
                 rep);
  else
    krylov_ops_t(c, n, A, M, static_cast<const double*>(b), ldb, static_cast<double*>(x), ldx,
                 nrhs, cfg, rep);
}

// The reduced-system operators on compact ReducedVectors:
// kind 0 matvec_lowrank, 1 matvec_otf (= matvec_exact with exact tips), 2
// apply_truncated_precond.  x, y: 2 k p x nrhs blocks, ld = ldr (full length).
template <class S>
void reduced_op_t(Fact* f, int kind, S* x, S* y, int nrhs) {
  if (f->Pg < 2) throw LrsError(LRS_ERR_PARAMETER, "reduced system needs p >= 2");
  if (kind != 1 && f->r == 0)
    throw LrsError(LRS_ERR_PARAMETER, "factorization has no low-rank spikes (n_svd = 0)");
  for (int c0 = 0; c0 < nrhs; c0 += MAX_RHS) {
    const int nr = std::min(MAX_RHS, nrhs - c0);
    S* xc = x + (int64_t)c0 * f->ldr;
    S* yc = y + (int64_t)c0 * f->ldr;
    if (kind == 0) {
      matvec_lowrank_t(f, xc, yc, nr);
    } else if (kind == 1) {
      DevBuf<S> z;
      z.alloc((size_t)f->n * nr);
      matvec_otf_t(f, xc, yc, z.get(), nr);
    } else {
      trunc_precond_t(f, xc, yc, nr);
    }
  }
}

// build_truncated_precond from explicit spikes: a factorization handle
// with no band factors whose "n-layout" is the compact reduced layout (partition i owns
// rows [2ki, 2k(i+1)): top tip, then bottom tip), so the interface setup and the
// reduced-system operators (apply_truncated_precond, matvec_lowrank) run unchanged.
// Spike arrays are device pointers: uT[i] (2k x r: the top then the bottom k-row tip of
// u of T_i, i < p-1), vT[i] (r x k), sT[i] (r); uW[i] (2k x r, tips of u of W_{i+1}),
// vW[i], sW[i].  apply_truncated_precond reads the bottom tips of T and the top tips of W,
// matvec_lowrank all four.
template <class S>
Fact* trunc_precond_t(Ctx* c, int64_t p, int64_t k, int r, const S* uTb, const S* vT,
                      const double* sT, const S* uWt, const S* vW, const double* sW) {
  std::unique_ptr<Fact> f(new Fact());
  constexpr int w = SW<S>;
  f->ctx = c;
  f->scalar = IsC<S>::value ? LRS_C128 : LRS_F64;
  f->sw = w;
  f->variant = LRS_VARIANT_T;
  f->P = f->Pg = (int)p;
  f->p0 = 0;
  f->k = k;
  f->n = 2 * k * p;
  f->ldr = f->n;
  f->row_lo = 0;
  f->row_hi = f->n;
  f->r = r;
  f->l = r;
  for (int64_t i = 0; i <= p; ++i) f->goff.push_back(2 * k * i);
  for (int64_t i = 0; i < p; ++i) {
    f->off.push_back(2 * k * i);
    f->size.push_back(2 * k);
    f->T.push_back(0);
    f->tbase.push_back(0);
    f->fbase.push_back(0);
  }
  upload(c, f->d_off, f->off);
  upload(c, f->d_size, f->size);
  upload(c, f->d_T, f->T);
  upload(c, f->d_goff, f->goff);
  upload(c, f->d_tbase, f->tbase);
  upload(c, f->d_fbase, f->fbase);
  const int64_t n = f->n, kr = k * r;
  f->uT.alloc((size_t)n * r * w);
  f->uW.alloc((size_t)n * r * w);
  f->vtT.alloc((size_t)p * kr * w);
  f->vtW.alloc((size_t)p * kr * w);
  f->sT.alloc((size_t)p * r);
  f->sW.alloc((size_t)p * r);
  for (DevBuf<double>* b : {&f->uT, &f->uW, &f->vtT, &f->vtW, &f->sT, &f->sW})
    LRS_CUDA(cudaMemsetAsync(b->get(), 0, b->bytes, c->stream));
  const size_t es = sizeof(S);
  for (int64_t i = 0; i + 1 < p; ++i) {
    // both u tips into the compact rows of their partition; v (r x k) transposed into
    // v^T (k x r) by a strided 2D copy
    LRS_CUDA(cudaMemcpy2DAsync(sp<S>(f->uT) + 2 * k * i, es * n, uTb + 2 * i * kr, es * 2 * k,
                               es * 2 * k, r, cudaMemcpyDeviceToDevice, c->stream));
    LRS_CUDA(cudaMemcpy2DAsync(sp<S>(f->uW) + 2 * k * (i + 1), es * n, uWt + 2 * i * kr,
                               es * 2 * k, es * 2 * k, r, cudaMemcpyDeviceToDevice, c->stream));
    for (int a = 0; a < r; ++a) {  // row a of v -> column a of v^T
      LRS_CUDA(cudaMemcpy2DAsync(sp<S>(f->vtT) + i * kr + (int64_t)a * k, es, vT + i * kr + a,
                                 es * r, es, k, cudaMemcpyDeviceToDevice, c->stream));
      LRS_CUDA(cudaMemcpy2DAsync(sp<S>(f->vtW) + (i + 1) * kr + (int64_t)a * k, es,
                                 vW + i * kr + a, es * r, es, k, cudaMemcpyDeviceToDevice,
                                 c->stream));
    }
    LRS_CUDA(cudaMemcpyAsync(f->sT.get() + i * r, sT + i * r, sizeof(double) * r,
                             cudaMemcpyDeviceToDevice, c->stream));
    LRS_CUDA(cudaMemcpyAsync(f->sW.get() + (i + 1) * r, sW + i * r, sizeof(double) * r,
                             cudaMemcpyDeviceToDevice, c->stream));
  }
  int bad_i = -1;
  double bad_c = 0.0;
  if (!finish_interfaces<S>(f.get(), r, &bad_i, &bad_c)) {
    LrsError e(LRS_ERR_ILL_CONDITIONED_INTERFACE,
               "interface " + std::to_string(bad_i) + " is ill-conditioned (cond_1 = " +
                   std::to_string(bad_c) + ")");
    e.iface = bad_i;
    e.cond = bad_c;
    throw e;
  }
  f->info.n = f->n;
  f->info.p = p;
  f->info.k = k;
  f->info.n_svd = r;
  f->info.l = r;
  f->info.variant = LRS_VARIANT_T;
  return f.release();
}

Fact* make_trunc_precond(Ctx* c, int32_t scalar, int64_t p, int64_t k, int r, const void* uTb,
                         const void* vT, const double* sT, const void* uWt, const void* vW,
                         const double* sW) {
  if (scalar == LRS_C128)
    return trunc_precond_t<zc>(c, p, k, r, static_cast<const zc*>(uTb), static_cast<const zc*>(vT),
                               sT, static_cast<const zc*>(uWt), static_cast<const zc*>(vW), sW);
  return trunc_precond_t<double>(c, p, k, r, static_cast<const double*>(uTb),
                                 static_cast<const double*>(vT), sT,
                                 static_cast<const double*>(uWt), static_cast<const double*>(vW),
                                 sW);
}

void reduced_op(Fact* f, int kind, void* x, void* y, int nrhs) {
  if (f->scalar == LRS_C128) reduced_op_t(f, kind, static_cast<zc*>(x), static_cast<zc*>(y), nrhs);
  else reduced_op_t(f, kind, static_cast<double*>(x), static_cast<double*>(y), nrhs);
}

void apply_precond(Fact* f, const void* in, int64_t ldi, void* out, int64_t ldo, int nrhs,
                   int mode) {
  if (f->scalar == LRS_C128)
    apply_variant_t(f, static_cast<const zc*>(in), ldi, static_cast<zc*>(out), ldo, nrhs, mode);
  else
    apply_variant_t(f, static_cast<const double*>(in), ldi, static_cast<double*>(out), ldo, nrhs,
                    mode);
}

}  // namespace lrs

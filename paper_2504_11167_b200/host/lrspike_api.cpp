// C++ drop-in API (include/lrspike/*.hpp) over the C-ABI of liblrspike_cuda.so.
//
// Every numerical operation is forwarded to the GPU library; this file moves host
// blocks, composes the SPEC operations out of C-ABI calls (randomized_spike_svd from
// the GPU band solves, SpMV, QR, Jacobi SVD and small GEMMs) and rethrows C-ABI statuses
// as the matching lrspike::Error subclass (errors.hpp).  Templated on the scalar (double,
// complex128) with explicit instantiations at the end.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>

#include "lrs_rng.h"
#include "lrspike/comm.hpp"
#include "lrspike/errors.hpp"
#include "lrspike/matrix.hpp"
#include "lrspike/solver.hpp"
#include "lrspike_capi.h"

namespace lrspike {

namespace {

[[noreturn]] void rethrow(lrs_status s, lrs_ctx* ctx) {
  lrs_error_info e{};
  lrs_last_error(ctx, &e);
  const std::string msg = e.message[0] ? e.message : lrs_status_string(s);
  switch (s) {
    case LRS_ERR_PARSE: throw ParseError(msg, (long)e.line);
    case LRS_ERR_UNSUPPORTED_FIELD: throw UnsupportedFieldError(msg);
    case LRS_ERR_DIMENSION: throw DimensionError(msg);
    case LRS_ERR_SINGULAR_SCALING: throw SingularScalingError(msg, (long)e.row);
    case LRS_ERR_LAYOUT: throw LayoutError(msg);
    case LRS_ERR_NOT_BLOCK_TRIDIAGONAL: throw NotBlockTridiagonalError(msg, (long)e.row, (long)e.col);
    case LRS_ERR_SINGULAR_BLOCK: throw SingularBlockError(msg, (long)e.column);
    case LRS_ERR_PARAMETER: throw ParameterError(msg);
    case LRS_ERR_ILL_CONDITIONED_INTERFACE:
      throw IllConditionedInterfaceError(msg, (int)e.interface_index, e.cond_estimate);
    case LRS_ERR_BREAKDOWN: throw BreakdownError(msg);
    case LRS_ERR_NOT_IMPLEMENTED: throw NotImplementedError(msg);
    case LRS_ERR_PRECOND_FAILURE: throw PreconditionerFailureError(msg);
    default: throw CudaError(msg);
  }
}

void check(lrs_status s, lrs_ctx* ctx) {
  if (s != LRS_OK) rethrow(s, ctx);
}

template <class S>
constexpr int32_t scalar_tag() {
  return is_complex<S>::value ? LRS_C128 : LRS_F64;
}

inline double conj_of(double a) { return a; }
inline complex128 conj_of(complex128 a) { return std::conj(a); }

// conjugate transpose of a host CSR (the adjoint coupling of the spike SVD)
template <class S>
CsrMatrixT<S> adjoint_of(const CsrMatrixT<S>& a) {
  CsrMatrixT<S> t = a.transposed();
  for (S& v : t.values) v = conj_of(v);
  return t;
}

lrs_iter_cfg to_c(Method m, int restart, double tol, index_t max_iters, double eps) {
  lrs_iter_cfg ic{};
  ic.method = m == Method::GMRES ? LRS_GMRES : m == Method::CG ? LRS_CG : LRS_BICGSTAB;
  ic.restart = restart;
  ic.tol = tol;
  ic.max_iters = max_iters;
  ic.breakdown_eps = eps;
  return ic;
}

SolveReport from_c(const lrs_report& r, const std::vector<double>& hist) {
  SolveReport rep;
  rep.converged = r.converged != 0;
  rep.breakdown = r.breakdown != 0;
  rep.iterations = r.iterations;
  rep.residual_history.assign(
      hist.begin(), hist.begin() + std::min<int64_t>(r.history_len, (int64_t)hist.size()));
  rep.precond_applications = r.precond_applications;
  rep.matvecs = r.matvecs;
  rep.ledger.reduced_matvec = {r.comm_messages[0], r.comm_scalars[0]};
  rep.ledger.precond_apply = {r.comm_messages[1], r.comm_scalars[1]};
  rep.ledger.recovery = {r.comm_messages[2], r.comm_scalars[2]};
  rep.comm_scalars = r.comm_scalars[0] + r.comm_scalars[1] + r.comm_scalars[2];
  rep.seed = r.seed;
  rep.wall_time = r.t_solve;
  rep.residual_final = r.residual_final;
  rep.inner_iterations = r.inner_iterations;
  rep.inner_solves = r.inner_solves;
  rep.comm_calls = r.comm_calls;
  rep.comm_host_syncs = r.comm_host_syncs;
  rep.scalar_syncs = r.scalar_syncs;
  return rep;
}

// a breakdown keeps the partial iterate: rethrow with it attached
template <class S>
[[noreturn]] void throw_breakdown(lrs_ctx* ctx, const DenseBlockT<S>& x, const SolveReport& rep) {
  lrs_error_info e{};
  lrs_last_error(ctx, &e);
  const double* p = reinterpret_cast<const double*>(x.data());
  const size_t nd = (size_t)x.size() * (is_complex<S>::value ? 2 : 1);
  throw BreakdownError(e.message[0] ? e.message : "BiCGStab breakdown",
                       std::vector<double>(p, p + nd), (long)x.rows(), (long)x.cols(),
                       is_complex<S>::value, rep.iterations);
}

}  // namespace

namespace detail {
// The device copy of a host CsrMatrixT made by spmv(): valid while the three arrays
// keep their storage and sizes (the SPEC makes a CsrMatrix immutable after construction).
struct DeviceCsrCache {
  lrs_mat* mat = nullptr;
  const void *rp = nullptr, *ci = nullptr, *va = nullptr;
  index_t n = -1, nnz = -1;
  ~DeviceCsrCache() {
    if (mat) lrs_mat_destroy(mat);
  }
};
}  // namespace detail

// ---- device objects ---------------------------------------------------------------------
Device::Device(int ordinal) { check(lrs_ctx_create(ordinal, nullptr, &h_), nullptr); }
Device::~Device() { lrs_ctx_destroy(h_); }
Device& Device::default_device() {
  // never destroyed: matrices and factorizations held in other statics may outlive it
  static Device* d = new Device(0);
  return *d;
}

template <class S>
DeviceMatrixT<S>::DeviceMatrixT(const CsrMatrixT<S>& a, Device& dev) : n_(a.n_rows), dev_(&dev) {
  if (!a.square()) throw DimensionError("the system matrix must be square");
  check(lrs_mat_upload_csr(dev.handle(), a.n_rows, a.nnz(), a.row_ptr.data(), a.col_idx.data(),
                           a.values.data(), scalar_tag<S>(), LRS_MEM_HOST, &h_),
        dev.handle());
}
template <class S>
DeviceMatrixT<S>::~DeviceMatrixT() {
  lrs_mat_destroy(h_);
}

template <class S>
DenseBlockT<S> DeviceMatrixT<S>::spmv(const DenseBlockT<S>& x) const {
  if (x.rows() != n_) throw DimensionError("spmv: A.n_cols must equal x.n_rows");
  DenseBlockT<S> y(n_, x.cols());
  check(lrs_spmv(h_, x.data(), n_, y.data(), n_, x.cols(), 0, LRS_MEM_HOST), dev_->handle());
  return y;
}

template <class S>
void DeviceMatrixT<S>::spmv_device(DeviceView<const S> x, DeviceView<S> y, bool accumulate) const {
  if (x.rows != n_ || y.rows != n_ || x.cols != y.cols)
    throw DimensionError("spmv: block shapes do not match A");
  check(lrs_spmv(h_, x.data, x.ld, y.data, y.ld, x.cols, accumulate ? 1 : 0, LRS_MEM_DEVICE),
        dev_->handle());
}

// spmv on a host CsrMatrixT: upload once, reuse the device copy while the arrays are unchanged
template <class S>
static lrs_mat* cached_device_csr(const CsrMatrixT<S>& a) {
  auto& c = a.device_cache;
  if (c && c->rp == a.row_ptr.data() && c->ci == a.col_idx.data() && c->va == a.values.data() &&
      c->n == a.n_rows && c->nnz == a.nnz())
    return c->mat;
  if (!a.square()) throw DimensionError("spmv: the matrix must be square");
  auto fresh = std::make_shared<detail::DeviceCsrCache>();
  lrs_ctx* ctx = Device::default_device().handle();
  check(lrs_mat_upload_csr(ctx, a.n_rows, a.nnz(), a.row_ptr.data(), a.col_idx.data(),
                           a.values.data(), scalar_tag<S>(), LRS_MEM_HOST, &fresh->mat),
        ctx);
  fresh->rp = a.row_ptr.data();
  fresh->ci = a.col_idx.data();
  fresh->va = a.values.data();
  fresh->n = a.n_rows;
  fresh->nnz = a.nnz();
  c = fresh;
  return c->mat;
}

template <class S>
DenseBlockT<S> spmv(const CsrMatrixT<S>& a, const DenseBlockT<S>& x) {
  if (a.n_cols != x.rows()) throw DimensionError("spmv: A.n_cols must equal x.n_rows");
  lrs_mat* m = cached_device_csr(a);
  DenseBlockT<S> y(a.n_rows, x.cols());
  check(lrs_spmv(m, x.data(), x.rows(), y.data(), y.rows(), x.cols(), 0, LRS_MEM_HOST),
        Device::default_device().handle());
  return y;
}

template <class S>
void spmv_accumulate(const CsrMatrixT<S>& a, const DenseBlockT<S>& x, DenseBlockT<S>& into) {
  if (a.n_cols != x.rows()) throw DimensionError("spmv: A.n_cols must equal x.n_rows");
  if (into.rows() != a.n_rows || into.cols() != x.cols())
    throw DimensionError("spmv: accumulator shape mismatch");
  lrs_mat* m = cached_device_csr(a);
  check(lrs_spmv(m, x.data(), x.rows(), into.data(), into.rows(), x.cols(), 1, LRS_MEM_HOST),
        Device::default_device().handle());
}

PartitionLayout make_layout(index_t n, index_t p, index_t k) {
  PartitionLayout l;
  l.p = p;
  l.k = k;
  l.sizes.assign(std::max<index_t>(p, 1), 0);
  check(lrs_make_layout(n, p, k, l.sizes.data()), nullptr);
  l.offsets.assign(std::max<index_t>(p, 1), 0);
  for (index_t i = 1; i < p; ++i) l.offsets[i] = l.offsets[i - 1] + l.sizes[i - 1];
  return l;
}

// ---- Communicator: the C view of a C++ transport -----------------------------------------
namespace {
int32_t comm_allgather(void* user, const double* send, double* recv, int64_t count) {
  try {
    static_cast<Communicator*>(user)->allgather(send, recv, count);
    return 0;
  } catch (...) {
    return 1;
  }
}
int32_t comm_sendrecv(void* user, const double* send, int64_t scount, int32_t dest, double* recv,
                      int64_t rcount, int32_t source) {
  try {
    static_cast<Communicator*>(user)->sendrecv(send, scount, dest, recv, rcount, source);
    return 0;
  } catch (...) {
    return 1;
  }
}
}  // namespace

const lrs_comm* Communicator::c_comm() {
  static_assert(sizeof(lrs_comm) <= sizeof(cstore_), "lrs_comm storage");
  lrs_comm c{};
  c.rank = rank();
  c.size = size();
  c.user = this;
  c.allgather = comm_allgather;
  c.sendrecv = comm_sendrecv;
  std::memcpy(cstore_.data(), &c, sizeof(c));
  return reinterpret_cast<const lrs_comm*>(cstore_.data());
}

std::array<unsigned char, 128> NcclCommunicator::nccl_unique_id() {
  std::array<unsigned char, 128> id{};
  check(lrs_comm_nccl_unique_id(id.data()), nullptr);
  return id;
}
NcclCommunicator::NcclCommunicator(Device& dev, const std::array<unsigned char, 128>& id, int rank,
                                   int size)
    : rank_(rank), size_(size) {
  check(lrs_comm_nccl_create(dev.handle(), id.data(), rank, size, &comm_), dev.handle());
}
NcclCommunicator::~NcclCommunicator() { lrs_comm_nccl_destroy(comm_); }
void NcclCommunicator::allgather(const double* send, double* recv, index_t count) {
  if (comm_->allgather(comm_->user, send, recv, count) != 0)
    throw CudaError("NCCL all-gather failed");
}
void NcclCommunicator::sendrecv(const double* send, index_t scount, int dest, double* recv,
                                index_t rcount, int source) {
  if (comm_->sendrecv(comm_->user, send, scount, dest, recv, rcount, source) != 0)
    throw CudaError("NCCL send/recv failed");
}

// ---- factorization ------------------------------------------------------------------------
template <class S>
static lrs_solver_cfg to_c(const SolverConfigT<S>& cfg) {
  lrs_solver_cfg c{};
  c.variant = cfg.variant == Variant::LR_SPIKE_T    ? LRS_VARIANT_T
              : cfg.variant == Variant::LR_SPIKE_I   ? LRS_VARIANT_I
              : cfg.variant == Variant::LR_SPIKE_OTF ? LRS_VARIANT_OTF
                                                     : LRS_VARIANT_BJ;
  c.inner_tol = cfg.inner_tol;
  c.inner_max_iters = cfg.inner_max_iters;
  c.otf_tol = cfg.otf_tol;
  c.otf_max_iters = cfg.otf_max_iters;
  c.otf_escalations = cfg.otf_escalations;
  c.factor_fp32 = cfg.factor_fp32 ? 1 : 0;
  c.spike_mode = cfg.spike_mode == SpikeMode::CouplingSvd ? LRS_SPIKE_COUPLING : LRS_SPIKE_SVD;
  c.passes = cfg.passes;
  c.p = cfg.p;
  c.k = cfg.k;
  c.n_svd = cfg.n_svd;
  c.oversample = cfg.oversample;
  c.seed = cfg.seed;
  return c;
}

template <class S>
SpikeFactorizationT<S>::SpikeFactorizationT(std::shared_ptr<DeviceMatrixT<S>> a,
                                            const SolverConfigT<S>& cfg, Communicator* comm)
    : a_(std::move(a)), cfg_(cfg) {
  const lrs_solver_cfg c = to_c(cfg);
  lrs_ctx* ctx = a_->device().handle();
  if (comm)
    check(lrs_factorize_dist(ctx, a_->handle(), &c, comm->c_comm(), &h_), ctx);
  else
    check(lrs_factorize(ctx, a_->handle(), &c, &h_), ctx);
  lrs_fact_info info{};
  lrs_fact_get_info(h_, &info);
  n_svd_ = info.n_svd;
  t_factorize_ = info.t_factorize;
  layout_.p = info.p;
  layout_.k = info.k;
  layout_.sizes.resize(info.p);
  layout_.offsets.resize(info.p);
  lrs_fact_get_layout(h_, layout_.sizes.data(), layout_.offsets.data());
  row_lo_ = 0;
  row_hi_ = a_->n();
  if (comm) {
    int64_t plo, phi, rlo, rhi;
    check(lrs_shard_plan(a_->n(), info.p, comm->size(), comm->rank(), &plo, &phi, &rlo, &rhi), ctx);
    row_lo_ = rlo;
    row_hi_ = rhi;
  }
}

template <class S>
SpikeFactorizationT<S>::~SpikeFactorizationT() {
  lrs_fact_destroy(h_);
}

template <class S>
CommLedger SpikeFactorizationT<S>::ledger() const {
  int64_t m[3], s[3];
  lrs_fact_get_ledger(h_, m, s);
  CommLedger l;
  l.reduced_matvec = {m[0], s[0]};
  l.precond_apply = {m[1], s[1]};
  l.recovery = {m[2], s[2]};
  return l;
}

template <class S>
static DenseBlockT<S> block_solve(const SpikeFactorizationT<S>& f, index_t i,
                                  const DenseBlockT<S>& rhs, int adjoint) {
  if (i < 0 || i >= f.layout().p) throw ParameterError("solve_block: no such partition");
  if (rhs.rows() != f.layout().sizes[i])
    throw DimensionError("solve_block: RHS rows must equal the block size");
  DenseBlockT<S> x(rhs.rows(), rhs.cols());
  check(lrs_solve_block(f.handle(), i, rhs.data(), rhs.rows(), x.data(), x.rows(), rhs.cols(),
                        adjoint, LRS_MEM_HOST),
        f.matrix()->device().handle());
  return x;
}

template <class S>
DenseBlockT<S> SpikeFactorizationT<S>::solve_block(index_t i, const DenseBlockT<S>& rhs) const {
  return block_solve(*this, i, rhs, 0);
}

template <class S>
DenseBlockT<S> SpikeFactorizationT<S>::solve_block_adjoint(index_t i, const DenseBlockT<S>& rhs) const {
  return block_solve(*this, i, rhs, 1);
}

template <class S>
LowRankSpikeT<S> SpikeFactorizationT<S>::spike(index_t i, Side side) const {
  LowRankSpikeT<S> s;
  s.side = side;
  s.u = DenseBlockT<S>(layout_.sizes.at(i), n_svd_);
  s.v = DenseBlockT<S>(n_svd_, layout_.k);
  s.sigma.assign(n_svd_, 0.0);
  check(lrs_fact_get_spike(h_, i, side == Side::T ? LRS_SIDE_T : LRS_SIDE_W,
                           reinterpret_cast<double*>(s.u.data()), s.sigma.data(),
                           reinterpret_cast<double*>(s.v.data())),
        a_->device().handle());
  for (double sg : s.sigma) s.rank_collapsed = s.rank_collapsed || sg == 0.0;
  return s;
}

template <class S>
void SpikeFactorizationT<S>::apply_device(DeviceView<const S> in, DeviceView<S> out) const {
  check(lrs_apply_precond(h_, in.data, in.ld, out.data, out.ld, in.cols, LRS_MEM_DEVICE),
        a_->device().handle());
}

template <class S>
std::shared_ptr<SpikeFactorizationT<S>> factorize(const CsrMatrixT<S>& a, const SolverConfigT<S>& cfg,
                                                  Device& dev) {
  return std::make_shared<SpikeFactorizationT<S>>(std::make_shared<DeviceMatrixT<S>>(a, dev), cfg);
}

template <class S>
std::shared_ptr<SpikeFactorizationT<S>> factorize_dist(const CsrMatrixT<S>& a,
                                                       const SolverConfigT<S>& cfg,
                                                       Communicator& comm, Device& dev) {
  return std::make_shared<SpikeFactorizationT<S>>(std::make_shared<DeviceMatrixT<S>>(a, dev), cfg,
                                                  &comm);
}

template <class S>
PartitionBlocksT<S> extract_blocks(const CsrMatrixT<S>& a, const PartitionLayout& lay) {
  if (!a.square()) throw DimensionError("extract_blocks: A must be square");
  const index_t p = lay.p, k = lay.k;
  if ((index_t)lay.sizes.size() != p ||
      std::accumulate(lay.sizes.begin(), lay.sizes.end(), index_t{0}) != a.n_rows)
    throw DimensionError("extract_blocks: layout does not match A");
  std::vector<index_t> off(p + 1, 0);
  for (index_t i = 0; i < p; ++i) off[i + 1] = off[i] + lay.sizes[i];
  struct Trip {
    std::vector<index_t> r, c;
    std::vector<S> v;
    void add(index_t rr, index_t cc, S vv) {
      r.push_back(rr);
      c.push_back(cc);
      v.push_back(vv);
    }
  };
  std::vector<Trip> tA(p), tB(p), tC(p);
  index_t part = 0;
  for (index_t row = 0; row < a.n_rows; ++row) {
    while (row >= off[part + 1]) ++part;
    const index_t lo = off[part], hi = off[part + 1];
    for (index_t q = a.row_ptr[row]; q < a.row_ptr[row + 1]; ++q) {
      const index_t col = a.col_idx[q];
      if (col >= lo && col < hi) {
        tA[part].add(row - lo, col - lo, a.values[q]);
      } else if (part + 1 < p && col >= hi && col < hi + k && row >= hi - k) {
        tB[part].add(row - (hi - k), col - hi, a.values[q]);  // bottom-left of the super block
      } else if (part > 0 && col < lo && col >= lo - k && row < lo + k) {
        tC[part].add(row - lo, col - (lo - k), a.values[q]);  // top-right of the sub block
      } else {
        throw NotBlockTridiagonalError("nonzero (" + std::to_string(row) + "," +
                                           std::to_string(col) +
                                           ") outside the block-tridiagonal pattern; increase k "
                                           "or decrease p",
                                       (long)row, (long)col);
      }
    }
  }
  PartitionBlocksT<S> out;
  out.layout = lay;
  for (index_t i = 0; i < p; ++i) {
    out.A.push_back(CsrMatrixT<S>::from_triplets(lay.sizes[i], lay.sizes[i], tA[i].r, tA[i].c, tA[i].v));
    out.B.push_back(i + 1 < p ? CsrMatrixT<S>::from_triplets(k, k, tB[i].r, tB[i].c, tB[i].v)
                              : CsrMatrixT<S>{});
    out.C.push_back(i > 0 ? CsrMatrixT<S>::from_triplets(k, k, tC[i].r, tC[i].c, tC[i].v)
                          : CsrMatrixT<S>{});
  }
  return out;
}

template <class S>
BlockFactorT<S> factorize_block(const CsrMatrixT<S>& a_i, Device& dev) {
  if (!a_i.square()) throw DimensionError("factorize_block: A_i must be square");
  SolverConfigT<S> cfg;
  cfg.variant = Variant::BLOCK_JACOBI;
  cfg.p = 1;
  cfg.k = 0;
  cfg.n_svd = 0;
  return BlockFactorT<S>(factorize(a_i, cfg, dev));
}

template <class S>
DenseBlockT<S> solve_block(const BlockFactorT<S>& f, const DenseBlockT<S>& rhs) {
  return f.factorization().solve_block(0, rhs);
}

template <class S>
DenseBlockT<S> solve_block_adjoint(const BlockFactorT<S>& f, const DenseBlockT<S>& rhs) {
  return f.factorization().solve_block_adjoint(0, rhs);
}

// ---- spikes: randomized_spike_svd composed from GPU operations -----------------------------
namespace {

template <class S>
struct Gpu {  // the dense building blocks on one context, host blocks in and out
  lrs_ctx* ctx;
  void qr(DenseBlockT<S>& A, DenseBlockT<S>* R) const {
    if (R) *R = DenseBlockT<S>(A.cols(), A.cols());
    check(lrs_dense_qr(ctx, scalar_tag<S>(), A.rows(), A.cols(), A.data(), A.rows(),
                       R ? R->data() : nullptr, LRS_MEM_HOST),
          ctx);
  }
  // R = U diag(sigma) V^H
  void svd(DenseBlockT<S> R, DenseBlockT<S>& U, DenseBlockT<S>& V, std::vector<double>& sg) const {
    const index_t l = R.rows();
    U = DenseBlockT<S>(l, l);
    V = DenseBlockT<S>(l, l);
    sg.assign(l, 0.0);
    check(lrs_dense_svd(ctx, scalar_tag<S>(), l, R.data(), U.data(), V.data(), sg.data(),
                        LRS_MEM_HOST),
          ctx);
  }
  // A (m x kk) * B[:, :ncols]
  DenseBlockT<S> gemm(const DenseBlockT<S>& A, const DenseBlockT<S>& B, index_t ncols,
                      bool conjC = false) const {
    DenseBlockT<S> C(A.rows(), ncols);
    check(lrs_dense_gemm(ctx, scalar_tag<S>(), A.rows(), ncols, A.cols(), A.data(), A.rows(),
                         B.data(), B.rows(), C.data(), C.rows(), conjC ? 1 : 0, LRS_MEM_HOST),
          ctx);
    return C;
  }
};

template <class S>
DenseBlockT<S> pad_rows(const DenseBlockT<S>& X, index_t n, Side side) {
  DenseBlockT<S> R(n, X.cols());
  const index_t r0 = side == Side::T ? n - X.rows() : 0;
  for (index_t c = 0; c < X.cols(); ++c)
    for (index_t i = 0; i < X.rows(); ++i) R(r0 + i, c) = X(i, c);
  return R;
}

template <class S>
DenseBlockT<S> first_cols(const DenseBlockT<S>& X, index_t nc) {
  DenseBlockT<S> o(X.rows(), nc);
  std::copy_n(X.data(), X.rows() * nc, o.data());
  return o;
}

template <class S>
DenseBlockT<S> scale_cols(DenseBlockT<S> X, const std::vector<double>& s) {
  for (index_t c = 0; c < X.cols(); ++c)
    for (index_t i = 0; i < X.rows(); ++i) X(i, c) *= s[c];
  return X;
}

template <class S>
DenseBlockT<S> transpose(const DenseBlockT<S>& X) {
  DenseBlockT<S> T(X.cols(), X.rows());
  for (index_t c = 0; c < X.cols(); ++c)
    for (index_t i = 0; i < X.rows(); ++i) T(c, i) = X(i, c);
  return T;
}

template <class S>
void finish_spike(LowRankSpikeT<S>& sp, index_t r) {
  const double s0 = sp.sigma.empty() ? 0.0 : sp.sigma[0];
  for (index_t j = 0; j < r; ++j)
    if (s0 == 0.0 || sp.sigma[j] < 1e-14 * s0) {  // truncate with the flag
      sp.sigma[j] = 0.0;
      sp.rank_collapsed = true;
    }
}

}  // namespace

template <class S>
LowRankSpikeT<S> randomized_spike_svd(const BlockFactorT<S>& F, const CsrMatrixT<S>& coupling,
                                      Side side, index_t n_svd, index_t oversample, int passes,
                                      std::uint64_t seed, index_t partition, SpikeMode mode) {
  const index_t k = coupling.n_rows, n = F.n();
  if (!coupling.square()) throw DimensionError("randomized_spike_svd: the coupling must be k x k");
  if (n < k) throw DimensionError("randomized_spike_svd: block smaller than k");
  if (oversample < 0) oversample = (n_svd + 1) / 2;
  const index_t l = n_svd + oversample;
  if (n_svd < 1 || n_svd > k) throw ParameterError("randomized_spike_svd: 1 <= n_svd <= k required");
  if (l > k || l > 96)
    throw ParameterError("randomized_spike_svd: n_svd + oversample <= min(k, 96) required");
  if (passes < 2) throw ParameterError("randomized_spike_svd: passes >= 2 required");
  const auto& fac = F.factorization();
  const Gpu<S> g{fac.matrix()->device().handle()};
  // Omega ~ N(0,1)^{k x l} from the stream (seed, partition, side)
  DenseBlockT<S> Om(k, l);
  const uint64_t key = lrs_rng_key(
      seed, LRS_STREAM_OMEGA + 2ull * (uint64_t)partition + (side == Side::W ? 1u : 0u));
  for (index_t e = 0; e < k * l; ++e) Om.data()[e] = S(lrs_rng_normal(key, (uint64_t)e));
  const CsrMatrixT<S> couplingH = adjoint_of(coupling);
  LowRankSpikeT<S> sp;
  sp.side = side;
  if (mode == SpikeMode::CouplingSvd) {  // the checker's coupling_spike_svd, step by step
    DenseBlockT<S> QB = spmv(coupling, first_cols(Om, n_svd));
    g.qr(QB, nullptr);
    for (int pi = 0; pi < (passes - 2) / 2; ++pi) {
      DenseBlockT<S> W = spmv(couplingH, QB);
      g.qr(W, nullptr);
      QB = spmv(coupling, W);
      g.qr(QB, nullptr);
    }
    DenseBlockT<S> Qz = spmv(couplingH, QB), R1, U1, V1;  // B^H Q_B = Q_z R_1
    std::vector<double> s1;
    g.qr(Qz, &R1);
    g.svd(R1, U1, V1, s1);  // R_1 = U_1 S_1 V_1^H  =>  B_r = (Q_B V_1) S_1 (Q_z U_1)^H
    const DenseBlockT<S> UBS = g.gemm(QB, scale_cols(V1, s1), n_svd);
    const DenseBlockT<S> VB = g.gemm(Qz, U1, n_svd);
    DenseBlockT<S> Y = fac.solve_block(0, pad_rows(UBS, n, side)), R2, U2, V2;
    g.qr(Y, &R2);
    g.svd(R2, U2, V2, sp.sigma);  // T~ = (Q_2 U_2) S_2 (V_B V_2)^H
    sp.u = g.gemm(Y, U2, n_svd);
    sp.v = transpose(g.gemm(VB, V2, n_svd, is_complex<S>::value));
    finish_spike(sp, n_svd);
    return sp;
  }
  auto T_apply = [&](const DenseBlockT<S>& X) {
    return fac.solve_block(0, pad_rows(spmv(coupling, X), n, side));
  };
  auto Tt_apply = [&](const DenseBlockT<S>& Q) {  // T^H Q = coupling^H (F^-H Q)|tip
    const DenseBlockT<S> Sx = fac.solve_block_adjoint(0, Q);
    return spmv(couplingH, Sx.middle_rows(side == Side::T ? n - k : 0, k));
  };
  DenseBlockT<S> Q = T_apply(Om);
  g.qr(Q, nullptr);
  for (int pi = 0; pi < (passes - 2) / 2; ++pi) {
    DenseBlockT<S> W = Tt_apply(Q);
    g.qr(W, nullptr);
    Q = T_apply(W);
    g.qr(Q, nullptr);
  }
  DenseBlockT<S> Zt = Tt_apply(Q), Rz, Ur, Vr;  // Zt = (Q^H T)^H = Q_z R_z
  g.qr(Zt, &Rz);
  std::vector<double> sg;
  g.svd(Rz, Ur, Vr, sg);  // R_z = U_R S V_R^H  =>  T ~ (Q V_R) S (Q_z U_R)^H
  sp.u = g.gemm(Q, Vr, n_svd);
  sp.v = transpose(g.gemm(Zt, Ur, n_svd, is_complex<S>::value));
  sp.sigma.assign(sg.begin(), sg.begin() + n_svd);
  finish_spike(sp, n_svd);
  return sp;
}

// ---- the reduced system ----------------------------------------------------------------
template <class S>
TruncatedPrecondT<S>::~TruncatedPrecondT() {
  lrs_fact_destroy(h_);
}

template <class S>
std::shared_ptr<TruncatedPrecondT<S>> build_truncated_precond(
    const std::vector<LowRankSpikeT<S>>& spT, const std::vector<LowRankSpikeT<S>>& spW, index_t k,
    Device& dev) {
  if (spT.empty() || spT.size() != spW.size())
    throw DimensionError("build_truncated_precond: p-1 spikes of each side required");
  const index_t p = (index_t)spT.size() + 1, r = (index_t)spT[0].sigma.size();
  std::vector<S> uT((size_t)(p - 1) * 2 * k * r), uW(uT.size());
  std::vector<S> vT((size_t)(p - 1) * k * r), vW(vT.size());
  std::vector<double> sT((size_t)(p - 1) * r), sW(sT.size());
  for (index_t i = 0; i + 1 < p; ++i) {
    const LowRankSpikeT<S>& t = spT[i];
    const LowRankSpikeT<S>& w = spW[i];
    if ((index_t)t.sigma.size() != r || (index_t)w.sigma.size() != r || t.v.cols() != k ||
        w.v.cols() != k || t.u.rows() < k || w.u.rows() < k)
      throw DimensionError("build_truncated_precond: spike shapes differ");
    for (int side = 0; side < 2; ++side) {  // [top tip; bottom tip], 2k x r per spike
      const LowRankSpikeT<S>& sp = side == 0 ? t : w;
      std::vector<S>& dst = side == 0 ? uT : uW;
      const auto tips = spike_tips(sp, k);
      for (index_t a = 0; a < r; ++a) {
        std::copy_n(tips.first.data() + a * k, k, dst.begin() + (i * r + a) * 2 * k);
        std::copy_n(tips.second.data() + a * k, k, dst.begin() + (i * r + a) * 2 * k + k);
      }
    }
    std::copy_n(t.v.data(), k * r, vT.begin() + i * k * r);
    std::copy_n(w.v.data(), k * r, vW.begin() + i * k * r);
    std::copy_n(t.sigma.begin(), r, sT.begin() + i * r);
    std::copy_n(w.sigma.begin(), r, sW.begin() + i * r);
  }
  lrs_fact* h = nullptr;
  check(lrs_trunc_precond_create(dev.handle(), scalar_tag<S>(), p, k, r, uT.data(), vT.data(),
                                 sT.data(), uW.data(), vW.data(), sW.data(), LRS_MEM_HOST, &h),
        dev.handle());
  return std::make_shared<TruncatedPrecondT<S>>(h, dev, p, k, r);
}

template <class S>
static ReducedVectorT<S> reduced(lrs_fact* h, lrs_ctx* ctx, int kind, const ReducedVectorT<S>& x) {
  ReducedVectorT<S> y(x.p, x.k, x.data.cols());
  check(lrs_reduced_apply(h, kind, x.data.data(), x.data.rows(), y.data.data(), y.data.rows(),
                          x.data.cols(), LRS_MEM_HOST),
        ctx);
  return y;
}

template <class S>
ReducedVectorT<S> apply_truncated_precond(const TruncatedPrecondT<S>& P, const ReducedVectorT<S>& g) {
  return reduced(P.handle(), P.device().handle(), LRS_REDUCED_TRUNC_PRECOND, g);
}
template <class S>
ReducedVectorT<S> matvec_lowrank(const TruncatedPrecondT<S>& P, const ReducedVectorT<S>& x) {
  return reduced(P.handle(), P.device().handle(), LRS_REDUCED_MATVEC_LOWRANK, x);
}
template <class S>
ReducedVectorT<S> matvec_lowrank(const SpikeFactorizationT<S>& f, const ReducedVectorT<S>& x) {
  return reduced(f.handle(), f.matrix()->device().handle(), LRS_REDUCED_MATVEC_LOWRANK, x);
}
template <class S>
ReducedVectorT<S> matvec_otf(const SpikeFactorizationT<S>& f, const ReducedVectorT<S>& x) {
  return reduced(f.handle(), f.matrix()->device().handle(), LRS_REDUCED_MATVEC_EXACT, x);
}

// ---- applies and solves ------------------------------------------------------------------
using ApplyFn = lrs_status (*)(lrs_fact*, const void*, int64_t, void*, int64_t, int64_t, int32_t);

template <class S>
static DenseBlockT<S> apply_impl(const SpikeFactorizationT<S>& f, const DenseBlockT<S>& rhs, ApplyFn fn) {
  if (rhs.rows() != f.matrix()->n()) throw DimensionError("apply: vector rows must equal n");
  DenseBlockT<S> x(rhs.rows(), rhs.cols());
  check(fn(f.handle(), rhs.data(), rhs.rows(), x.data(), x.rows(), rhs.cols(), LRS_MEM_HOST),
        f.matrix()->device().handle());
  return x;
}

template <class S>
DenseBlockT<S> apply_precond_T(const SpikeFactorizationT<S>& f, const DenseBlockT<S>& rhs) {
  return apply_impl(f, rhs, lrs_apply_precond_T);
}
template <class S>
DenseBlockT<S> apply_precond_I(const SpikeFactorizationT<S>& f, const DenseBlockT<S>& rhs) {
  if (f.config().variant != Variant::LR_SPIKE_I)
    throw ParameterError("apply_precond_I needs an LR_SPIKE_I factorization");
  return apply_impl(f, rhs, lrs_apply_precond);
}
template <class S>
DenseBlockT<S> apply_block_jacobi(const SpikeFactorizationT<S>& f, const DenseBlockT<S>& rhs) {
  return apply_impl(f, rhs, lrs_apply_block_jacobi);
}

template <class S>
std::pair<DenseBlockT<S>, SolveReport> solve(const CsrMatrixT<S>& a, const DenseBlockT<S>& rhs,
                                             const SolverConfigT<S>& cfg,
                                             std::shared_ptr<SpikeFactorizationT<S>> f) {
  if (!f) f = factorize(a, cfg);
  if (rhs.rows() != a.n_rows) throw DimensionError("solve: rhs rows must equal n");
  const IterConfigT<S>& it = cfg.outer;
  lrs_iter_cfg ic = to_c(it.method, it.restart, it.tol, it.max_iters, it.breakdown_eps);
  if (it.initial_guess) {
    if (it.initial_guess->rows() != rhs.rows() || it.initial_guess->cols() != rhs.cols())
      throw DimensionError("initial guess shape must match the rhs");
    ic.x0 = it.initial_guess->data();
  }
  std::vector<double> hist(1 << 16);
  lrs_report r{};
  r.history = hist.data();
  r.history_cap = (int64_t)hist.size();
  DenseBlockT<S> x(rhs.rows(), rhs.cols());
  lrs_ctx* ctx = f->matrix()->device().handle();
  const lrs_status s = lrs_solve(f->handle(), f->matrix()->handle(), rhs.data(), rhs.rows(),
                                 x.data(), x.rows(), rhs.cols(), &ic, &r, LRS_MEM_HOST);
  SolveReport rep = from_c(r, hist);
  if (s == LRS_ERR_BREAKDOWN) throw_breakdown(ctx, x, rep);
  check(s, ctx);
  return {std::move(x), std::move(rep)};
}

// ---- Krylov drivers on operators ------------------------------------------------------------
namespace {
template <class S>
struct OpCtx {
  const LinearOperatorT<S>* op;
  index_t n;
};
template <class S>
int32_t op_tramp(void* user, const void* in, void* out, int64_t ld, int64_t n_rhs) {
  auto* c = static_cast<OpCtx<S>*>(user);
  try {
    (*c->op)(DeviceView<const S>{static_cast<const S*>(in), c->n, n_rhs, ld},
             DeviceView<S>{static_cast<S*>(out), c->n, n_rhs, ld});
    return 0;
  } catch (...) {
    return 1;
  }
}

template <class S>
std::pair<DenseBlockT<S>, SolveReport> krylov(Method m, const LinearOperatorT<S>& A,
                                              const LinearOperatorT<S>* M, const DenseBlockT<S>& b,
                                              const IterConfigT<S>& it, Device& dev) {
  const index_t n = b.rows();
  OpCtx<S> ca{&A, n}, cm{M, n};
  lrs_operator oa{&ca, op_tramp<S>}, om{&cm, op_tramp<S>};
  lrs_iter_cfg ic = to_c(m, it.restart, it.tol, it.max_iters, it.breakdown_eps);
  if (it.initial_guess) {
    if (it.initial_guess->rows() != n || it.initial_guess->cols() != b.cols())
      throw DimensionError("initial guess shape must match the rhs");
    ic.x0 = it.initial_guess->data();
  }
  std::vector<double> hist(1 << 16);
  lrs_report r{};
  r.history = hist.data();
  r.history_cap = (int64_t)hist.size();
  DenseBlockT<S> x(n, b.cols());
  const lrs_status s = lrs_krylov(dev.handle(), n, scalar_tag<S>(), &oa, M ? &om : nullptr,
                                  b.data(), n, x.data(), n, b.cols(), &ic, &r, LRS_MEM_HOST);
  SolveReport rep = from_c(r, hist);
  if (s == LRS_ERR_BREAKDOWN) throw_breakdown(dev.handle(), x, rep);
  check(s, dev.handle());
  return {std::move(x), std::move(rep)};
}
}  // namespace

template <class S>
LinearOperatorT<S> as_operator(const DeviceMatrixT<S>& a) {
  return [&a](DeviceView<const S> in, DeviceView<S> out) { a.spmv_device(in, out); };
}
template <class S>
LinearOperatorT<S> as_operator(const SpikeFactorizationT<S>& f) {
  return [&f](DeviceView<const S> in, DeviceView<S> out) { f.apply_device(in, out); };
}
template <class S>
std::pair<DenseBlockT<S>, SolveReport> bicgstab(const LinearOperatorT<S>& A, const LinearOperatorT<S>* M,
                                                const DenseBlockT<S>& b, const IterConfigT<S>& it,
                                                Device& dev) {
  return krylov(Method::BICGSTAB, A, M, b, it, dev);
}
template <class S>
std::pair<DenseBlockT<S>, SolveReport> cg(const LinearOperatorT<S>& A, const LinearOperatorT<S>* M,
                                          const DenseBlockT<S>& b, const IterConfigT<S>& it,
                                          Device& dev) {
  return krylov(Method::CG, A, M, b, it, dev);
}
template <class S>
std::pair<DenseBlockT<S>, SolveReport> gmres(const LinearOperatorT<S>& A, const LinearOperatorT<S>* M,
                                             const DenseBlockT<S>& b, const IterConfigT<S>& it,
                                             Device& dev) {
  return krylov(Method::GMRES, A, M, b, it, dev);
}

// ---- explicit instantiations: double (the reference's CsrMatrix) and complex128 ---------
#define LRS_INSTANTIATE(S)                                                                        \
  template class DeviceMatrixT<S>;                                                                \
  template class SpikeFactorizationT<S>;                                                          \
  template class TruncatedPrecondT<S>;                                                            \
  template DenseBlockT<S> spmv(const CsrMatrixT<S>&, const DenseBlockT<S>&);                      \
  template void spmv_accumulate(const CsrMatrixT<S>&, const DenseBlockT<S>&, DenseBlockT<S>&);    \
  template PartitionBlocksT<S> extract_blocks(const CsrMatrixT<S>&, const PartitionLayout&);      \
  template BlockFactorT<S> factorize_block(const CsrMatrixT<S>&, Device&);                        \
  template DenseBlockT<S> solve_block(const BlockFactorT<S>&, const DenseBlockT<S>&);             \
  template DenseBlockT<S> solve_block_adjoint(const BlockFactorT<S>&, const DenseBlockT<S>&);     \
  template LowRankSpikeT<S> randomized_spike_svd(const BlockFactorT<S>&, const CsrMatrixT<S>&,    \
                                                 Side, index_t, index_t, int, std::uint64_t,      \
                                                 index_t, SpikeMode);                             \
  template std::shared_ptr<TruncatedPrecondT<S>> build_truncated_precond(                         \
      const std::vector<LowRankSpikeT<S>>&, const std::vector<LowRankSpikeT<S>>&, index_t,         \
      Device&);                                                                                   \
  template ReducedVectorT<S> apply_truncated_precond(const TruncatedPrecondT<S>&,                 \
                                                     const ReducedVectorT<S>&);                   \
  template ReducedVectorT<S> matvec_lowrank(const TruncatedPrecondT<S>&, const ReducedVectorT<S>&); \
  template ReducedVectorT<S> matvec_lowrank(const SpikeFactorizationT<S>&,                        \
                                            const ReducedVectorT<S>&);                            \
  template ReducedVectorT<S> matvec_otf(const SpikeFactorizationT<S>&, const ReducedVectorT<S>&); \
  template std::shared_ptr<SpikeFactorizationT<S>> factorize(const CsrMatrixT<S>&,                \
                                                             const SolverConfigT<S>&, Device&);   \
  template std::shared_ptr<SpikeFactorizationT<S>> factorize_dist(                                \
      const CsrMatrixT<S>&, const SolverConfigT<S>&, Communicator&, Device&);                     \
  template DenseBlockT<S> apply_precond_T(const SpikeFactorizationT<S>&, const DenseBlockT<S>&);  \
  template DenseBlockT<S> apply_precond_I(const SpikeFactorizationT<S>&, const DenseBlockT<S>&);  \
  template DenseBlockT<S> apply_block_jacobi(const SpikeFactorizationT<S>&, const DenseBlockT<S>&); \
  template std::pair<DenseBlockT<S>, SolveReport> solve(                                          \
      const CsrMatrixT<S>&, const DenseBlockT<S>&, const SolverConfigT<S>&,                       \
      std::shared_ptr<SpikeFactorizationT<S>>);                                                   \
  template LinearOperatorT<S> as_operator(const DeviceMatrixT<S>&);                               \
  template LinearOperatorT<S> as_operator(const SpikeFactorizationT<S>&);                         \
  template std::pair<DenseBlockT<S>, SolveReport> bicgstab(                                       \
      const LinearOperatorT<S>&, const LinearOperatorT<S>*, const DenseBlockT<S>&,                \
      const IterConfigT<S>&, Device&);                                                            \
  template std::pair<DenseBlockT<S>, SolveReport> cg(const LinearOperatorT<S>&,                   \
                                                     const LinearOperatorT<S>*,                   \
                                                     const DenseBlockT<S>&,                       \
                                                     const IterConfigT<S>&, Device&);             \
  template std::pair<DenseBlockT<S>, SolveReport> gmres(                                          \
      const LinearOperatorT<S>&, const LinearOperatorT<S>*, const DenseBlockT<S>&,                \
      const IterConfigT<S>&, Device&);
LRS_INSTANTIATE(double)
LRS_INSTANTIATE(complex128)
#undef LRS_INSTANTIATE

}  // namespace lrspike

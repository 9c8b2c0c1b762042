// C++ drop-in API (include/lrspike/*.hpp) over the C-ABI of liblrspike_cuda.so.
//
// Host containers (CsrMatrix, DenseBlock) and their structural helpers
// mirror reference proj/core/src/matrix.cpp; every numerical operation is
// forwarded to the GPU library, and C-ABI statuses are rethrown as the
// matching lrspike::Error subclass (errors.hpp).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

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

}  // namespace

// ---- CsrMatrix (host structure; matrix.cpp semantics) ---------------------------------
double CsrMatrix::coeff(index_t row, index_t col) const {
  const auto b = col_idx.begin() + row_ptr[row], e = col_idx.begin() + row_ptr[row + 1];
  const auto it = std::lower_bound(b, e, col);
  return (it == e || *it != col) ? 0.0 : values[static_cast<size_t>(it - col_idx.begin())];
}

void CsrMatrix::validate() const {
  if (n_rows < 0 || n_cols < 0) throw DimensionError("negative dimension");
  if (static_cast<index_t>(row_ptr.size()) != n_rows + 1)
    throw DimensionError("row_ptr length must be n_rows + 1");
  if (row_ptr.front() != 0) throw DimensionError("row_ptr[0] must be 0");
  if (row_ptr.back() != nnz()) throw DimensionError("row_ptr[n_rows] must equal nnz");
  if (col_idx.size() != values.size()) throw DimensionError("col_idx/values length mismatch");
  for (index_t i = 0; i < n_rows; ++i) {
    if (row_ptr[i] > row_ptr[i + 1]) throw DimensionError("row_ptr must be non-decreasing");
    for (index_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      if (col_idx[p] < 0 || col_idx[p] >= n_cols) throw DimensionError("column index out of range");
      if (p > row_ptr[i] && col_idx[p] <= col_idx[p - 1])
        throw DimensionError("column indices must be strictly increasing within a row");
    }
  }
}

DenseBlock CsrMatrix::to_dense() const {
  DenseBlock d(n_rows, n_cols);
  for (index_t i = 0; i < n_rows; ++i)
    for (index_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) d(i, col_idx[p]) = values[p];
  return d;
}

CsrMatrix CsrMatrix::transposed() const {
  CsrMatrix t;
  t.n_rows = n_cols;
  t.n_cols = n_rows;
  t.row_ptr.assign(n_cols + 1, 0);
  for (index_t p = 0; p < nnz(); ++p) ++t.row_ptr[col_idx[p] + 1];
  std::partial_sum(t.row_ptr.begin(), t.row_ptr.end(), t.row_ptr.begin());
  t.col_idx.resize(nnz());
  t.values.resize(nnz());
  std::vector<index_t> next(t.row_ptr.begin(), t.row_ptr.end() - 1);
  for (index_t i = 0; i < n_rows; ++i)
    for (index_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const index_t q = next[col_idx[p]]++;
      t.col_idx[q] = i;
      t.values[q] = values[p];
    }
  return t;
}

CsrMatrix CsrMatrix::from_triplets(index_t n_rows, index_t n_cols, std::vector<index_t> rows,
                                   std::vector<index_t> cols, std::vector<double> vals) {
  if (rows.size() != cols.size() || rows.size() != vals.size())
    throw DimensionError("triplet arrays must have equal length");
  std::vector<size_t> order(rows.size());
  std::iota(order.begin(), order.end(), size_t{0});
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b];
  });
  CsrMatrix m;
  m.n_rows = n_rows;
  m.n_cols = n_cols;
  m.row_ptr.assign(n_rows + 1, 0);
  index_t last_r = -1, last_c = -1;
  for (size_t s : order) {
    if (rows[s] < 0 || rows[s] >= n_rows || cols[s] < 0 || cols[s] >= n_cols)
      throw DimensionError("triplet index out of range");
    if (rows[s] == last_r && cols[s] == last_c) {  // duplicate in ANY row: summed
      m.values.back() += vals[s];
      continue;
    }
    m.col_idx.push_back(cols[s]);
    m.values.push_back(vals[s]);
    ++m.row_ptr[rows[s] + 1];
    last_r = rows[s];
    last_c = cols[s];
  }
  std::partial_sum(m.row_ptr.begin(), m.row_ptr.end(), m.row_ptr.begin());
  m.validate();
  return m;
}

CsrMatrix CsrMatrix::identity(index_t n) {
  CsrMatrix m;
  m.n_rows = m.n_cols = n;
  m.row_ptr.resize(n + 1);
  m.col_idx.resize(n);
  m.values.assign(n, 1.0);
  std::iota(m.row_ptr.begin(), m.row_ptr.end(), index_t{0});
  std::iota(m.col_idx.begin(), m.col_idx.end(), index_t{0});
  return m;
}

BandMetrics band_metrics(const CsrMatrix& a) {
  if (!a.square()) throw DimensionError("band_metrics: matrix must be square");
  BandMetrics m;
  double dsum = 0.0, tsum = 0.0;
  for (index_t i = 0; i < a.n_rows; ++i)
    for (index_t p = a.row_ptr[i]; p < a.row_ptr[i + 1]; ++p) {
      const index_t j = a.col_idx[p];
      if (j > i) m.band.upper_half_bw = std::max(m.band.upper_half_bw, j - i);
      if (j < i) m.band.lower_half_bw = std::max(m.band.lower_half_bw, i - j);
      tsum += std::fabs(a.values[p]);
      if (i == j) dsum += std::fabs(a.values[p]);
    }
  m.band.k = std::max(m.band.upper_half_bw, m.band.lower_half_bw);
  m.diag_weight = tsum > 0.0 ? dsum / tsum : 0.0;
  const double cells = double(m.band.upper_half_bw + m.band.lower_half_bw + 1) * double(a.n_rows);
  m.band_density = cells > 0.0 ? double(a.nnz()) / cells : 0.0;
  return m;
}

// ---- device objects ---------------------------------------------------------------------
Device::Device(int ordinal) { check(lrs_ctx_create(ordinal, nullptr, &h_), nullptr); }
Device::~Device() { lrs_ctx_destroy(h_); }
Device& Device::default_device() {
  static Device d(0);
  return d;
}

DeviceMatrix::DeviceMatrix(const CsrMatrix& a, Device& dev) : n_(a.n_rows), dev_(&dev) {
  if (!a.square()) throw DimensionError("the system matrix must be square");
  check(lrs_mat_upload_csr(dev.handle(), a.n_rows, a.nnz(), a.row_ptr.data(), a.col_idx.data(),
                           a.values.data(), LRS_F64, LRS_MEM_HOST, &h_),
        dev.handle());
}
DeviceMatrix::~DeviceMatrix() { lrs_mat_destroy(h_); }

DenseBlock DeviceMatrix::spmv(const DenseBlock& x) const {
  if (x.rows() != n_) throw DimensionError("spmv: A.n_cols must equal x.n_rows");
  DenseBlock y(n_, x.cols());
  check(lrs_spmv(h_, x.data(), n_, y.data(), n_, x.cols(), 0, LRS_MEM_HOST), dev_->handle());
  return y;
}

DenseBlock spmv(const CsrMatrix& a, const DenseBlock& x) {
  if (a.n_cols != x.rows()) throw DimensionError("spmv: A.n_cols must equal x.n_rows");
  DeviceMatrix d(a);
  return d.spmv(x);
}

void spmv_accumulate(const CsrMatrix& a, const DenseBlock& x, DenseBlock& into) {
  if (a.n_cols != x.rows()) throw DimensionError("spmv: A.n_cols must equal x.n_rows");
  if (into.rows() != a.n_rows || into.cols() != x.cols())
    throw DimensionError("spmv: accumulator shape mismatch");
  DeviceMatrix d(a);
  check(lrs_spmv(d.handle(), x.data(), x.rows(), into.data(), into.rows(), x.cols(), 1,
                 LRS_MEM_HOST),
        d.device().handle());
}

PartitionLayout make_layout(index_t n, index_t p, index_t k) {
  PartitionLayout l;
  l.p = p;
  l.k = k;
  l.sizes.assign(std::max<index_t>(p, 1), 0);
  check(lrs_make_layout(n, p, k, l.sizes.data()), nullptr);
  l.offsets.assign(p, 0);
  for (index_t i = 1; i < p; ++i) l.offsets[i] = l.offsets[i - 1] + l.sizes[i - 1];
  return l;
}

SpikeFactorization::SpikeFactorization(std::shared_ptr<DeviceMatrix> a, const SolverConfig& cfg)
    : a_(std::move(a)), cfg_(cfg) {
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
  lrs_ctx* ctx = a_->device().handle();
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
}

SpikeFactorization::~SpikeFactorization() { lrs_fact_destroy(h_); }

CommLedger SpikeFactorization::ledger() const {
  int64_t m[3], s[3];
  lrs_fact_get_ledger(h_, m, s);
  CommLedger l;
  l.reduced_matvec = {m[0], s[0]};
  l.precond_apply = {m[1], s[1]};
  l.recovery = {m[2], s[2]};
  return l;
}

DenseBlock SpikeFactorization::solve_block(index_t i, const DenseBlock& rhs) const {
  if (i < 0 || i >= layout_.p) throw ParameterError("no such partition");
  if (rhs.rows() != layout_.sizes[i]) throw DimensionError("solve_block: RHS rows must equal the block size");
  DenseBlock x(rhs.rows(), rhs.cols());
  check(lrs_solve_block(h_, i, rhs.data(), rhs.rows(), x.data(), x.rows(), rhs.cols(), 0,
                        LRS_MEM_HOST),
        a_->device().handle());
  return x;
}

DenseBlock SpikeFactorization::solve_block_adjoint(index_t i, const DenseBlock& rhs) const {
  if (i < 0 || i >= layout_.p) throw ParameterError("no such partition");
  if (rhs.rows() != layout_.sizes[i]) throw DimensionError("solve_block: RHS rows must equal the block size");
  DenseBlock x(rhs.rows(), rhs.cols());
  check(lrs_solve_block(h_, i, rhs.data(), rhs.rows(), x.data(), x.rows(), rhs.cols(), 1,
                        LRS_MEM_HOST),
        a_->device().handle());
  return x;
}

void SpikeFactorization::spike(index_t i, int side, DenseBlock& u, std::vector<double>& sigma,
                               DenseBlock& v) const {
  u = DenseBlock(layout_.sizes.at(i), n_svd_);
  v = DenseBlock(n_svd_, layout_.k);
  sigma.assign(n_svd_, 0.0);
  check(lrs_fact_get_spike(h_, i, side, u.data(), sigma.data(), v.data()), a_->device().handle());
}

std::shared_ptr<SpikeFactorization> factorize(const CsrMatrix& a, const SolverConfig& cfg) {
  return std::make_shared<SpikeFactorization>(std::make_shared<DeviceMatrix>(a), cfg);
}

PartitionBlocks extract_blocks(const CsrMatrix& a, const PartitionLayout& lay) {
  if (!a.square()) throw DimensionError("extract_blocks: A must be square");
  index_t total = 0;
  for (index_t s : lay.sizes) total += s;
  if (total != a.n_rows || (index_t)lay.sizes.size() != lay.p)
    throw DimensionError("extract_blocks: layout does not match A");
  const index_t p = lay.p, k = lay.k;
  std::vector<index_t> off(p + 1, 0);
  for (index_t i = 0; i < p; ++i) off[i + 1] = off[i] + lay.sizes[i];
  struct Trip {
    std::vector<index_t> r, c;
    std::vector<double> v;
  };
  std::vector<Trip> tA(p), tB(p), tC(p);
  index_t part = 0;
  for (index_t row = 0; row < a.n_rows; ++row) {
    while (row >= off[part + 1]) ++part;
    for (index_t q = a.row_ptr[row]; q < a.row_ptr[row + 1]; ++q) {
      const index_t col = a.col_idx[q];
      const double v = a.values[q];
      if (col >= off[part] && col < off[part + 1]) {
        tA[part].r.push_back(row - off[part]);
        tA[part].c.push_back(col - off[part]);
        tA[part].v.push_back(v);
      } else if (part + 1 < p && col >= off[part + 1] && col < off[part + 1] + k &&
                 row >= off[part + 1] - k) {  // B_part: bottom-left k x k of the super block
        tB[part].r.push_back(row - (off[part + 1] - k));
        tB[part].c.push_back(col - off[part + 1]);
        tB[part].v.push_back(v);
      } else if (part > 0 && col < off[part] && col >= off[part] - k && row < off[part] + k) {
        tC[part].r.push_back(row - off[part]);  // C_part: top-right k x k of the sub block
        tC[part].c.push_back(col - (off[part] - k));
        tC[part].v.push_back(v);
      } else {
        throw NotBlockTridiagonalError("nonzero (" + std::to_string(row) + "," +
                                           std::to_string(col) +
                                           ") outside the block-tridiagonal pattern; increase k "
                                           "or decrease p",
                                       (long)row, (long)col);
      }
    }
  }
  PartitionBlocks out;
  out.layout = lay;
  for (index_t i = 0; i < p; ++i) {
    out.A.push_back(CsrMatrix::from_triplets(lay.sizes[i], lay.sizes[i], tA[i].r, tA[i].c, tA[i].v));
    out.B.push_back(i + 1 < p ? CsrMatrix::from_triplets(k, k, tB[i].r, tB[i].c, tB[i].v)
                              : CsrMatrix{});
    out.C.push_back(i > 0 ? CsrMatrix::from_triplets(k, k, tC[i].r, tC[i].c, tC[i].v)
                          : CsrMatrix{});
  }
  return out;
}

index_t BlockFactor::n() const { return f_->layout().sizes.at(0); }

BlockFactor factorize_block(const CsrMatrix& a_i) {
  if (!a_i.square()) throw DimensionError("factorize_block: A_i must be square");
  SolverConfig cfg;
  cfg.variant = Variant::BLOCK_JACOBI;
  cfg.p = 1;
  cfg.k = 0;
  cfg.n_svd = 0;
  return BlockFactor(factorize(a_i, cfg));
}

DenseBlock solve_block(const BlockFactor& f, const DenseBlock& rhs) {
  return f.factorization().solve_block(0, rhs);
}

DenseBlock solve_block_adjoint(const BlockFactor& f, const DenseBlock& rhs) {
  return f.factorization().solve_block_adjoint(0, rhs);
}

using ApplyFn = lrs_status (*)(lrs_fact*, const void*, int64_t, void*, int64_t, int64_t, int32_t);

static DenseBlock apply_impl(const SpikeFactorization& f, const DenseBlock& rhs, ApplyFn fn) {
  if (rhs.rows() != f.matrix()->n()) throw DimensionError("apply: vector rows must equal n");
  DenseBlock x(rhs.rows(), rhs.cols());
  lrs_ctx* ctx = f.matrix()->device().handle();
  check(fn(f.handle(), rhs.data(), rhs.rows(), x.data(), x.rows(), rhs.cols(), LRS_MEM_HOST), ctx);
  return x;
}

DenseBlock apply_precond_T(const SpikeFactorization& f, const DenseBlock& rhs) {
  return apply_impl(f, rhs, lrs_apply_precond_T);
}

DenseBlock apply_precond_I(const SpikeFactorization& f, const DenseBlock& rhs) {
  if (f.config().variant != Variant::LR_SPIKE_I)
    throw ParameterError("apply_precond_I needs an LR_SPIKE_I factorization");
  return apply_impl(f, rhs, lrs_apply_precond);
}

DenseBlock apply_block_jacobi(const SpikeFactorization& f, const DenseBlock& rhs) {
  return apply_impl(f, rhs, lrs_apply_block_jacobi);
}

std::pair<DenseBlock, SolveReport> solve(const CsrMatrix& a, const DenseBlock& rhs,
                                         const SolverConfig& cfg,
                                         std::shared_ptr<SpikeFactorization> f) {
  if (!f) f = factorize(a, cfg);
  if (rhs.rows() != a.n_rows) throw DimensionError("solve: rhs rows must equal n");
  const IterConfig& it = cfg.outer;
  lrs_iter_cfg ic{};
  ic.method = it.method == Method::GMRES ? LRS_GMRES
              : it.method == Method::CG  ? LRS_CG
                                         : LRS_BICGSTAB;
  ic.restart = it.restart;
  ic.tol = it.tol;
  ic.max_iters = it.max_iters;
  ic.breakdown_eps = it.breakdown_eps;
  if (it.initial_guess) {
    if (it.initial_guess->rows() != rhs.rows() || it.initial_guess->cols() != rhs.cols())
      throw DimensionError("initial guess shape must match the rhs");
    ic.x0 = it.initial_guess->data();
  }
  std::vector<double> hist(1 << 16);
  lrs_report r{};
  r.history = hist.data();
  r.history_cap = (int64_t)hist.size();
  DenseBlock x(rhs.rows(), rhs.cols());
  lrs_ctx* ctx = f->matrix()->device().handle();
  const lrs_status s = lrs_solve(f->handle(), f->matrix()->handle(), rhs.data(), rhs.rows(),
                                 x.data(), x.rows(), rhs.cols(), &ic, &r, LRS_MEM_HOST);
  SolveReport rep;
  rep.converged = r.converged != 0;
  rep.iterations = r.iterations;
  rep.residual_history.assign(hist.begin(), hist.begin() + r.history_len);
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
  check(s, ctx);
  return {std::move(x), std::move(rep)};
}

}  // namespace lrspike

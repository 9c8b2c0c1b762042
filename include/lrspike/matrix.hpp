// lrspike sparse_core of the C++ drop-in API: host containers + GPU spmv.
//
// Names and semantics of reference proj/core/include/lrspike/matrix.hpp (Apache-2.0, the
// interface this library replaces): index_t, DenseBlock (column-major, (row, col)
// indexing), CsrMatrix with coeff / validate / to_dense / transposed / from_triplets /
// identity, spmv, spmv_accumulate, BandInfo, BandMetrics, band_metrics.  The containers
// are templated on the scalar (the config-5 FEAST systems are complex128);
// CsrMatrix / DenseBlock are the double instances the reference names, CsrMatrixZ /
// DenseBlockZ the complex128 ones.  Eigen is not part of this build, so DenseBlockT is an
// in-house column-major block (SPEC.md:30 permits any layout).  spmv runs on the GPU
// through the C-ABI (include/lrspike_capi.h); there is no host arithmetic path.
#pragma once

#include <algorithm>
#include <complex>
#include <cstdint>
#include <memory>
#include <numeric>
#include <type_traits>
#include <vector>

#include "lrspike/errors.hpp"

namespace lrspike {

using index_t = std::int64_t;
using complex128 = std::complex<double>;

template <class S>
struct is_complex : std::false_type {};
template <>
struct is_complex<complex128> : std::true_type {};

/// Dense multi-column block, column-major, (row, col) indexing.
template <class S>
class DenseBlockT {
 public:
  using scalar_type = S;
  DenseBlockT() = default;
  DenseBlockT(index_t rows, index_t cols)
      : rows_(rows), cols_(cols), v_(static_cast<size_t>(rows * cols), S(0)) {}
  static DenseBlockT Zero(index_t rows, index_t cols) { return DenseBlockT(rows, cols); }
  static DenseBlockT Identity(index_t n) {
    DenseBlockT d(n, n);
    for (index_t i = 0; i < n; ++i) d(i, i) = S(1);
    return d;
  }
  index_t rows() const { return rows_; }
  index_t cols() const { return cols_; }
  index_t size() const { return rows_ * cols_; }
  S& operator()(index_t r, index_t c) { return v_[static_cast<size_t>(r + c * rows_)]; }
  const S& operator()(index_t r, index_t c) const { return v_[static_cast<size_t>(r + c * rows_)]; }
  S* data() { return v_.data(); }
  const S* data() const { return v_.data(); }
  /// Rows [r0, r0 + n) of every column, as a new block.
  DenseBlockT middle_rows(index_t r0, index_t n) const {
    DenseBlockT o(n, cols_);
    for (index_t c = 0; c < cols_; ++c)
      std::copy_n(v_.begin() + (r0 + c * rows_), n, o.v_.begin() + c * n);
    return o;
  }

 private:
  index_t rows_ = 0, cols_ = 0;
  std::vector<S> v_;
};

using DenseBlock = DenseBlockT<double>;
using DenseBlockZ = DenseBlockT<complex128>;

namespace detail {
struct DeviceCsrCache;  // the device copy behind spmv(const CsrMatrixT&), see spmv below
}

/// General sparse matrix in compressed-row form (reference matrix.hpp:17-48 invariants:
/// row_ptr non-decreasing from 0 to nnz, column indices in range and strictly increasing
/// within a row).  Immutable after construction by contract.
template <class S>
struct CsrMatrixT {
  using scalar_type = S;
  index_t n_rows = 0;
  index_t n_cols = 0;
  std::vector<index_t> row_ptr;
  std::vector<index_t> col_idx;
  std::vector<S> values;
  /// Device copy made by the first spmv() on this matrix, reused while the arrays are
  /// the same (same storage, sizes); copies of the matrix share it.
  mutable std::shared_ptr<detail::DeviceCsrCache> device_cache;

  index_t nnz() const { return static_cast<index_t>(values.size()); }
  bool square() const { return n_rows == n_cols; }

  /// Entry (row, col), zero when not stored (binary search within the row).
  S coeff(index_t row, index_t col) const {
    const auto first = col_idx.begin() + row_ptr[row];
    const auto last = col_idx.begin() + row_ptr[row + 1];
    const auto hit = std::lower_bound(first, last, col);
    if (hit == last || *hit != col) return S(0);
    return values[static_cast<size_t>(hit - col_idx.begin())];
  }

  /// Throws DimensionError on the first violated structural invariant.
  void validate() const {
    if (n_rows < 0 || n_cols < 0) throw DimensionError("CsrMatrix: negative dimension");
    if (static_cast<index_t>(row_ptr.size()) != n_rows + 1)
      throw DimensionError("CsrMatrix: row_ptr must hold n_rows + 1 offsets");
    if (col_idx.size() != values.size())
      throw DimensionError("CsrMatrix: col_idx and values differ in length");
    if (row_ptr.front() != 0 || row_ptr.back() != nnz())
      throw DimensionError("CsrMatrix: row_ptr must run from 0 to nnz");
    for (index_t i = 0; i < n_rows; ++i) {
      const index_t b = row_ptr[i], e = row_ptr[i + 1];
      if (e < b) throw DimensionError("CsrMatrix: row_ptr decreases at row " + std::to_string(i));
      for (index_t q = b; q < e; ++q) {
        const index_t j = col_idx[q];
        if (j < 0 || j >= n_cols)
          throw DimensionError("CsrMatrix: column index out of range in row " + std::to_string(i));
        if (q > b && j <= col_idx[q - 1])
          throw DimensionError("CsrMatrix: columns not strictly increasing in row " +
                               std::to_string(i));
      }
    }
  }

  DenseBlockT<S> to_dense() const {
    DenseBlockT<S> d(n_rows, n_cols);
    for (index_t i = 0; i < n_rows; ++i)
      for (index_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) d(i, col_idx[q]) = values[q];
    return d;
  }

  /// A^T (plain transpose; the adjoint couplings conjugate on the device).
  CsrMatrixT transposed() const {
    CsrMatrixT t;
    t.n_rows = n_cols;
    t.n_cols = n_rows;
    std::vector<index_t> count(n_cols + 1, 0);
    for (index_t j : col_idx) ++count[j + 1];
    std::partial_sum(count.begin(), count.end(), count.begin());
    t.row_ptr = count;
    t.col_idx.resize(col_idx.size());
    t.values.resize(values.size());
    for (index_t i = 0; i < n_rows; ++i)  // rows in order: each t row stays sorted
      for (index_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
        const index_t dst = count[col_idx[q]]++;
        t.col_idx[dst] = i;
        t.values[dst] = values[q];
      }
    return t;
  }

  /// CSR from unsorted (row, col, value) triplets.  Duplicates are summed in every row
  /// (the documented contract, SPEC.md:43 / :75; DESIGN.md records the reference's
  /// first-row-only bug).
  static CsrMatrixT from_triplets(index_t n_rows, index_t n_cols, std::vector<index_t> rows,
                                  std::vector<index_t> cols, std::vector<S> vals) {
    if (rows.size() != cols.size() || rows.size() != vals.size())
      throw DimensionError("from_triplets: rows, cols and vals differ in length");
    for (size_t t = 0; t < rows.size(); ++t)
      if (rows[t] < 0 || rows[t] >= n_rows || cols[t] < 0 || cols[t] >= n_cols)
        throw DimensionError("from_triplets: index out of range");
    std::vector<size_t> perm(rows.size());
    std::iota(perm.begin(), perm.end(), size_t{0});
    std::stable_sort(perm.begin(), perm.end(), [&](size_t a, size_t b) {
      return rows[a] < rows[b] || (rows[a] == rows[b] && cols[a] < cols[b]);
    });
    CsrMatrixT m;
    m.n_rows = n_rows;
    m.n_cols = n_cols;
    m.row_ptr.assign(static_cast<size_t>(n_rows + 1), 0);
    for (size_t t = 0; t < perm.size(); ++t) {
      const size_t s = perm[t];
      const bool dup = t > 0 && rows[perm[t - 1]] == rows[s] && cols[perm[t - 1]] == cols[s];
      if (dup) {
        m.values.back() += vals[s];
      } else {
        m.col_idx.push_back(cols[s]);
        m.values.push_back(vals[s]);
        ++m.row_ptr[rows[s] + 1];
      }
    }
    std::partial_sum(m.row_ptr.begin(), m.row_ptr.end(), m.row_ptr.begin());
    m.validate();
    return m;
  }

  static CsrMatrixT identity(index_t n) {
    CsrMatrixT m;
    m.n_rows = m.n_cols = n;
    m.row_ptr.resize(static_cast<size_t>(n + 1));
    std::iota(m.row_ptr.begin(), m.row_ptr.end(), index_t{0});
    m.col_idx.resize(static_cast<size_t>(n));
    std::iota(m.col_idx.begin(), m.col_idx.end(), index_t{0});
    m.values.assign(static_cast<size_t>(n), S(1));
    return m;
  }
};

using CsrMatrix = CsrMatrixT<double>;
using CsrMatrixZ = CsrMatrixT<complex128>;

/// y = A x on the GPU, columns visited in ascending order per row (reference
/// matrix.cpp:121-136).  The first call uploads A (validate, int32 device indices, A^T)
/// and keeps the device copy in A.device_cache; later calls on the same (unmodified)
/// matrix reuse it.
template <class S>
DenseBlockT<S> spmv(const CsrMatrixT<S>& a, const DenseBlockT<S>& x);
/// into += A x on the GPU.
template <class S>
void spmv_accumulate(const CsrMatrixT<S>& a, const DenseBlockT<S>& x, DenseBlockT<S>& into);

struct BandInfo {
  index_t upper_half_bw = 0;
  index_t lower_half_bw = 0;
  index_t k = 0;  // max(upper, lower): the coupling half-bandwidth SPEC.md:201 suggests
};

struct BandMetrics {
  BandInfo band;
  double diag_weight = 0.0;   // sum |a_ii| / sum |a_ij|
  double band_density = 0.0;  // nnz / ((ku + kl + 1) n)
};

template <class S>
BandMetrics band_metrics(const CsrMatrixT<S>& a) {
  if (!a.square()) throw DimensionError("band_metrics: matrix must be square");
  BandMetrics m;
  double on_diag = 0.0, total = 0.0;
  for (index_t i = 0; i < a.n_rows; ++i)
    for (index_t q = a.row_ptr[i]; q < a.row_ptr[i + 1]; ++q) {
      const index_t d = a.col_idx[q] - i;
      m.band.upper_half_bw = std::max(m.band.upper_half_bw, d);
      m.band.lower_half_bw = std::max(m.band.lower_half_bw, -d);
      const double mag = std::abs(a.values[q]);
      total += mag;
      if (d == 0) on_diag += mag;
    }
  m.band.k = std::max(m.band.upper_half_bw, m.band.lower_half_bw);
  m.diag_weight = total > 0.0 ? on_diag / total : 0.0;
  const double cells =
      static_cast<double>(m.band.upper_half_bw + m.band.lower_half_bw + 1) * static_cast<double>(a.n_rows);
  m.band_density = cells > 0.0 ? static_cast<double>(a.nnz()) / cells : 0.0;
  return m;
}

}  // namespace lrspike

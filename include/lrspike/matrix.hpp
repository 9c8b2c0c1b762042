// lrspike sparse_core of the C++ drop-in API (host containers + GPU spmv).
//
// Same names and signatures as reference proj/core/include/lrspike/matrix.hpp:
// index_t, DenseBlock (column-major, (row, col) indexing -- an in-house class
// here because Eigen is not part of this build), CsrMatrix with coeff /
// validate / to_dense / transposed / from_triplets / identity, spmv,
// spmv_accumulate, BandInfo, BandMetrics, band_metrics.  spmv runs on the GPU
// through the C-ABI (include/lrspike_capi.h); there is no host arithmetic path.
#pragma once

#include <cstdint>
#include <vector>

namespace lrspike {

using index_t = std::int64_t;

/// Dense multi-column block, column-major, (row, col) indexing.
class DenseBlock {
 public:
  DenseBlock() = default;
  DenseBlock(index_t rows, index_t cols) : rows_(rows), cols_(cols), v_(rows * cols, 0.0) {}
  static DenseBlock Zero(index_t rows, index_t cols) { return DenseBlock(rows, cols); }
  static DenseBlock Identity(index_t n) {
    DenseBlock d(n, n);
    for (index_t i = 0; i < n; ++i) d(i, i) = 1.0;
    return d;
  }
  index_t rows() const { return rows_; }
  index_t cols() const { return cols_; }
  index_t size() const { return rows_ * cols_; }
  double& operator()(index_t r, index_t c) { return v_[r + c * rows_]; }
  double operator()(index_t r, index_t c) const { return v_[r + c * rows_]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

 private:
  index_t rows_ = 0, cols_ = 0;
  std::vector<double> v_;
};

/// General sparse matrix in compressed-row form (matrix.hpp:17-48 invariants).
struct CsrMatrix {
  index_t n_rows = 0;
  index_t n_cols = 0;
  std::vector<index_t> row_ptr;
  std::vector<index_t> col_idx;
  std::vector<double> values;

  index_t nnz() const { return static_cast<index_t>(values.size()); }
  bool square() const { return n_rows == n_cols; }
  double coeff(index_t row, index_t col) const;
  /// Throws DimensionError on any violated structural invariant.
  void validate() const;
  DenseBlock to_dense() const;
  CsrMatrix transposed() const;
  /// Builds a CSR from unsorted triplets; duplicates are summed in every row
  /// (the documented contract, SPEC.md:43/:75 -- see DESIGN.md on the reference bug).
  static CsrMatrix from_triplets(index_t n_rows, index_t n_cols, std::vector<index_t> rows,
                                 std::vector<index_t> cols, std::vector<double> vals);
  static CsrMatrix identity(index_t n);
};

/// y = A * x on the GPU (ascending column order per row, matrix.cpp:121-136).
DenseBlock spmv(const CsrMatrix& a, const DenseBlock& x);
/// into += A * x on the GPU.
void spmv_accumulate(const CsrMatrix& a, const DenseBlock& x, DenseBlock& into);

struct BandInfo {
  index_t upper_half_bw = 0;
  index_t lower_half_bw = 0;
  index_t k = 0;
};

struct BandMetrics {
  BandInfo band;
  double diag_weight = 0.0;
  double band_density = 0.0;
};

BandMetrics band_metrics(const CsrMatrix& a);

}  // namespace lrspike

// Matrix Market ingestion and the reorder pipeline (include/lrspike/reorder.hpp), plus the
// extern "C" layer of include/lrspike_io.h for FFI callers.  SPEC.md:39-47 (io) and
// SPEC.md:96-133 (reorder); host-side structural preprocessing ahead of the GPU solver.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <functional>
#include <fstream>
#include <numeric>
#include <sstream>
#include <string>

#include "lrspike/errors.hpp"
#include "lrspike/reorder.hpp"
#include "lrspike_io.h"

namespace lrspike {

namespace {

std::string lower(std::string s) {
  for (auto& ch : s) ch = (char)std::tolower((unsigned char)ch);
  return s;
}

}  // namespace

CsrMatrix read_matrix_market(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open " + path, 0);
  std::string line;
  long ln = 0;
  if (!std::getline(in, line)) throw ParseError("empty file", 1);
  ++ln;
  std::istringstream hs(line);
  std::string banner, object, format, field, symmetry;
  hs >> banner >> object >> format >> field >> symmetry;
  if (banner != "%%MatrixMarket" || lower(object) != "matrix")
    throw ParseError("missing %%MatrixMarket matrix header", ln);
  format = lower(format);
  field = lower(field);
  symmetry = lower(symmetry);
  if (format != "coordinate") throw UnsupportedFieldError("only the coordinate format is supported");
  if (field == "complex" || symmetry == "hermitian")
    throw UnsupportedFieldError("complex Matrix Market field is not supported (real scalars)");
  if (field != "real" && field != "integer" && field != "pattern" && field != "double")
    throw ParseError("unknown field '" + field + "'", ln);
  if (symmetry != "general" && symmetry != "symmetric" && symmetry != "skew-symmetric")
    throw ParseError("unknown symmetry '" + symmetry + "'", ln);
  const bool pattern = field == "pattern";
  long long nr = -1, nc = -1, nz = -1;
  while (std::getline(in, line)) {
    ++ln;
    if (line.empty() || line[0] == '%') continue;
    std::istringstream ss(line);
    if (!(ss >> nr >> nc >> nz) || nr < 0 || nc < 0 || nz < 0)
      throw ParseError("malformed size line", ln);
    break;
  }
  if (nz < 0) throw ParseError("missing size line", ln);
  std::vector<index_t> rows, cols;
  std::vector<double> vals;
  rows.reserve(nz * (symmetry == "general" ? 1 : 2));
  cols.reserve(rows.capacity());
  vals.reserve(rows.capacity());
  long long got = 0;
  while (got < nz && std::getline(in, line)) {
    ++ln;
    if (line.empty() || line[0] == '%') continue;
    std::istringstream ss(line);
    long long i, j;
    double v = 1.0;
    if (!(ss >> i >> j) || (!pattern && !(ss >> v)))
      throw ParseError("malformed entry", ln);
    if (i < 1 || i > nr || j < 1 || j > nc) throw ParseError("entry index out of range", ln);
    if (!std::isfinite(v)) throw ParseError("non-finite value", ln);
    rows.push_back(i - 1);
    cols.push_back(j - 1);
    vals.push_back(v);
    if (symmetry != "general" && i != j) {
      rows.push_back(j - 1);
      cols.push_back(i - 1);
      vals.push_back(symmetry == "skew-symmetric" ? -v : v);
    }
    ++got;
  }
  if (got < nz) throw ParseError("expected " + std::to_string(nz) + " entries, found " +
                                     std::to_string(got), ln + 1);
  return CsrMatrix::from_triplets(nr, nc, std::move(rows), std::move(cols), std::move(vals));
}

void write_matrix_market(const std::string& path, const CsrMatrix& a) {
  a.validate();
  FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw DimensionError("cannot write " + path);
  std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
  std::fprintf(f, "%lld %lld %lld\n", (long long)a.n_rows, (long long)a.n_cols, (long long)a.nnz());
  for (index_t r = 0; r < a.n_rows; ++r)
    for (index_t p = a.row_ptr[r]; p < a.row_ptr[r + 1]; ++p)
      std::fprintf(f, "%lld %lld %.17g\n", (long long)r + 1, (long long)a.col_idx[p] + 1,
                   a.values[p]);
  std::fclose(f);
}

Permutation Permutation::identity(index_t n) {
  Permutation p;
  p.forward.resize(n);
  std::iota(p.forward.begin(), p.forward.end(), index_t{0});
  p.inverse = p.forward;
  return p;
}

Permutation Permutation::from_order(const std::vector<index_t>& order) {
  Permutation p;
  const index_t n = (index_t)order.size();
  p.inverse = order;
  p.forward.assign(n, -1);
  for (index_t k = 0; k < n; ++k) {
    if (order[k] < 0 || order[k] >= n || p.forward[order[k]] >= 0)
      throw DimensionError("permutation is not a bijection");
    p.forward[order[k]] = k;
  }
  return p;
}

std::pair<CsrMatrix, std::vector<index_t>> strip_disconnected(const CsrMatrix& a) {
  if (!a.square()) throw DimensionError("strip_disconnected: matrix must be square");
  const index_t n = a.n_rows;
  std::vector<char> linked(n, 0);
  for (index_t r = 0; r < n; ++r)
    for (index_t p = a.row_ptr[r]; p < a.row_ptr[r + 1]; ++p)
      if (a.col_idx[p] != r) linked[r] = linked[a.col_idx[p]] = 1;
  std::vector<index_t> keep, removed, newidx(n, -1);
  for (index_t i = 0; i < n; ++i) {
    if (linked[i]) {
      newidx[i] = (index_t)keep.size();
      keep.push_back(i);
    } else {
      removed.push_back(i);
    }
  }
  CsrMatrix b;
  b.n_rows = b.n_cols = (index_t)keep.size();
  b.row_ptr.assign(b.n_rows + 1, 0);
  for (index_t k = 0; k < b.n_rows; ++k) {
    const index_t r = keep[k];
    for (index_t p = a.row_ptr[r]; p < a.row_ptr[r + 1]; ++p)
      if (newidx[a.col_idx[p]] >= 0) {
        b.col_idx.push_back(newidx[a.col_idx[p]]);
        b.values.push_back(a.values[p]);
      }
    b.row_ptr[k + 1] = (index_t)b.col_idx.size();
  }
  return {std::move(b), std::move(removed)};
}

std::pair<CsrMatrix, std::vector<double>> diagonal_scale(const CsrMatrix& a) {
  if (!a.square()) throw DimensionError("diagonal_scale: matrix must be square");
  const index_t n = a.n_rows;
  std::vector<double> d(n, 0.0);
  for (index_t r = 0; r < n; ++r) {
    const double v = a.coeff(r, r);
    if (v == 0.0)
      throw SingularScalingError("zero diagonal entry in row " + std::to_string(r) +
                                     " (structural zero diagonals are rejected, not repaired)",
                                 (long)r);
    d[r] = 1.0 / std::sqrt(std::fabs(v));
  }
  CsrMatrix b = a;
  for (index_t r = 0; r < n; ++r)
    for (index_t p = b.row_ptr[r]; p < b.row_ptr[r + 1]; ++p)
      b.values[p] = d[r] * a.values[p] * d[b.col_idx[p]];
  return {std::move(b), std::move(d)};
}

Permutation rcm_ordering(const CsrMatrix& a) {
  if (!a.square()) throw DimensionError("rcm_ordering: matrix must be square");
  const index_t n = a.n_rows;
  // adjacency of the pattern of A + A^T without the diagonal, neighbours sorted by index
  std::vector<std::vector<index_t>> adj(n);
  for (index_t r = 0; r < n; ++r)
    for (index_t p = a.row_ptr[r]; p < a.row_ptr[r + 1]; ++p) {
      const index_t c = a.col_idx[p];
      if (c != r) {
        adj[r].push_back(c);
        adj[c].push_back(r);
      }
    }
  std::vector<index_t> deg(n);
  for (index_t v = 0; v < n; ++v) {
    auto& l = adj[v];
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
    deg[v] = (index_t)l.size();
  }
  auto by_deg = [&](index_t x, index_t y) { return deg[x] != deg[y] ? deg[x] < deg[y] : x < y; };
  std::vector<index_t> level(n, -1), order;
  order.reserve(n);
  std::vector<char> placed(n, 0);
  // BFS levels from v within its component: returns (eccentricity, last level's vertices)
  auto bfs_levels = [&](index_t v, std::vector<index_t>& comp) {
    comp.clear();
    comp.push_back(v);
    level[v] = 0;
    index_t ecc = 0;
    for (size_t h = 0; h < comp.size(); ++h) {
      const index_t u = comp[h];
      for (index_t w : adj[u])
        if (level[w] < 0) {
          level[w] = level[u] + 1;
          ecc = std::max(ecc, level[w]);
          comp.push_back(w);
        }
    }
    std::vector<index_t> last;
    for (index_t u : comp)
      if (level[u] == ecc) last.push_back(u);
    for (index_t u : comp) level[u] = -1;
    return std::make_pair(ecc, last);
  };
  std::vector<index_t> comp;
  for (index_t s = 0; s < n; ++s) {
    if (placed[s]) continue;
    // George-Liu pseudo-peripheral vertex, starting from the lowest vertex of the component
    index_t v = s;
    auto [ecc, last] = bfs_levels(v, comp);
    while (true) {
      const index_t u = *std::min_element(last.begin(), last.end(), by_deg);
      auto [e2, l2] = bfs_levels(u, comp);
      if (e2 <= ecc) break;
      v = u;
      ecc = e2;
      last = l2;
    }
    // Cuthill-McKee from v: neighbours by ascending (degree, index)
    std::deque<index_t> q{v};
    placed[v] = 1;
    while (!q.empty()) {
      const index_t u = q.front();
      q.pop_front();
      order.push_back(u);
      std::vector<index_t> nb;
      for (index_t w : adj[u])
        if (!placed[w]) nb.push_back(w);
      std::sort(nb.begin(), nb.end(), by_deg);
      for (index_t w : nb) {
        placed[w] = 1;
        q.push_back(w);
      }
    }
  }
  std::reverse(order.begin(), order.end());
  return Permutation::from_order(order);
}

CsrMatrix apply_permutation(const CsrMatrix& a, const Permutation& rowp, const Permutation& colp) {
  if ((index_t)rowp.forward.size() != a.n_rows || (index_t)colp.forward.size() != a.n_cols)
    throw DimensionError("apply_permutation: permutation size does not match the matrix");
  std::vector<index_t> r, c;
  std::vector<double> v;
  r.reserve(a.nnz());
  c.reserve(a.nnz());
  v.reserve(a.nnz());
  for (index_t i = 0; i < a.n_rows; ++i)
    for (index_t p = a.row_ptr[i]; p < a.row_ptr[i + 1]; ++p) {
      r.push_back(rowp.forward[i]);
      c.push_back(colp.forward[a.col_idx[p]]);
      v.push_back(a.values[p]);
    }
  return CsrMatrix::from_triplets(a.n_rows, a.n_cols, std::move(r), std::move(c), std::move(v));
}

}  // namespace lrspike

// ---------------------------------------------------------------------------------------
// extern "C" layer (include/lrspike_io.h)
// ---------------------------------------------------------------------------------------
using namespace lrspike;

namespace {

thread_local lrs_io_error g_io_err{};

int32_t io_guard(const std::function<void()>& fn) {
  g_io_err = lrs_io_error{};
  try {
    fn();
    return LRS_OK;
  } catch (const ParseError& e) {
    g_io_err.line = e.line();
    std::snprintf(g_io_err.message, sizeof(g_io_err.message), "%s", e.what());
    return LRS_ERR_PARSE;
  } catch (const UnsupportedFieldError& e) {
    std::snprintf(g_io_err.message, sizeof(g_io_err.message), "%s", e.what());
    return LRS_ERR_UNSUPPORTED_FIELD;
  } catch (const SingularScalingError& e) {
    g_io_err.row = e.row();
    std::snprintf(g_io_err.message, sizeof(g_io_err.message), "%s", e.what());
    return LRS_ERR_SINGULAR_SCALING;
  } catch (const DimensionError& e) {
    std::snprintf(g_io_err.message, sizeof(g_io_err.message), "%s", e.what());
    return LRS_ERR_DIMENSION;
  } catch (const std::exception& e) {
    std::snprintf(g_io_err.message, sizeof(g_io_err.message), "%s", e.what());
    return LRS_ERR_PARAMETER;
  }
}

CsrMatrix from_host(const lrs_csr_host* a) {
  CsrMatrix m;
  m.n_rows = a->n_rows;
  m.n_cols = a->n_cols;
  m.row_ptr.assign(a->row_ptr, a->row_ptr + a->n_rows + 1);
  m.col_idx.assign(a->col_idx, a->col_idx + a->nnz);
  m.values.assign(a->values, a->values + a->nnz);
  m.validate();
  return m;
}

void to_host(const CsrMatrix& m, lrs_csr_host* out) {
  out->n_rows = m.n_rows;
  out->n_cols = m.n_cols;
  out->nnz = m.nnz();
  out->row_ptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (m.n_rows + 1)));
  out->col_idx = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<index_t>(1, m.nnz())));
  out->values = static_cast<double*>(std::malloc(sizeof(double) * std::max<index_t>(1, m.nnz())));
  if (!out->row_ptr || !out->col_idx || !out->values) throw std::bad_alloc();
  std::copy(m.row_ptr.begin(), m.row_ptr.end(), out->row_ptr);
  std::copy(m.col_idx.begin(), m.col_idx.end(), out->col_idx);
  std::copy(m.values.begin(), m.values.end(), out->values);
}

}  // namespace

extern "C" {

int32_t lrs_io_read_mm(const char* path, lrs_csr_host* out) {
  if (!path || !out) return LRS_ERR_PARAMETER;
  return io_guard([&] { to_host(read_matrix_market(path), out); });
}

int32_t lrs_io_write_mm(const char* path, const lrs_csr_host* a) {
  if (!path || !a) return LRS_ERR_PARAMETER;
  return io_guard([&] { write_matrix_market(path, from_host(a)); });
}

void lrs_io_free(lrs_csr_host* a) {
  if (!a) return;
  std::free(a->row_ptr);
  std::free(a->col_idx);
  std::free(a->values);
  a->row_ptr = a->col_idx = nullptr;
  a->values = nullptr;
}

int32_t lrs_reorder_rcm(const lrs_csr_host* a, int64_t* forward) {
  if (!a || !forward) return LRS_ERR_PARAMETER;
  return io_guard([&] {
    const Permutation p = rcm_ordering(from_host(a));
    std::copy(p.forward.begin(), p.forward.end(), forward);
  });
}

int32_t lrs_reorder_strip(const lrs_csr_host* a, lrs_csr_host* out, int64_t* removed,
                          int64_t* n_removed) {
  if (!a || !out || !removed || !n_removed) return LRS_ERR_PARAMETER;
  return io_guard([&] {
    auto [b, rem] = strip_disconnected(from_host(a));
    to_host(b, out);
    std::copy(rem.begin(), rem.end(), removed);
    *n_removed = (int64_t)rem.size();
  });
}

int32_t lrs_reorder_scale(const lrs_csr_host* a, lrs_csr_host* out, double* scale) {
  if (!a || !out || !scale) return LRS_ERR_PARAMETER;
  return io_guard([&] {
    auto [b, d] = diagonal_scale(from_host(a));
    to_host(b, out);
    std::copy(d.begin(), d.end(), scale);
  });
}

int32_t lrs_reorder_permute(const lrs_csr_host* a, const int64_t* row_forward,
                            const int64_t* col_forward, lrs_csr_host* out) {
  if (!a || !row_forward || !col_forward || !out) return LRS_ERR_PARAMETER;
  return io_guard([&] {
    std::vector<index_t> rf(row_forward, row_forward + a->n_rows);
    std::vector<index_t> cf(col_forward, col_forward + a->n_cols);
    std::vector<index_t> ri(a->n_rows), ci(a->n_cols);
    for (index_t i = 0; i < a->n_rows; ++i) ri[i] = i;
    Permutation rp, cp;
    std::vector<index_t> ro(a->n_rows, -1), co(a->n_cols, -1);
    for (index_t i = 0; i < a->n_rows; ++i) {
      if (rf[i] < 0 || rf[i] >= a->n_rows || ro[rf[i]] >= 0)
        throw DimensionError("row permutation is not a bijection");
      ro[rf[i]] = i;
    }
    for (index_t j = 0; j < a->n_cols; ++j) {
      if (cf[j] < 0 || cf[j] >= a->n_cols || co[cf[j]] >= 0)
        throw DimensionError("column permutation is not a bijection");
      co[cf[j]] = j;
    }
    rp = Permutation::from_order(ro);
    cp = Permutation::from_order(co);
    to_host(apply_permutation(from_host(a), rp, cp), out);
  });
}

int32_t lrs_io_last_error(lrs_io_error* out) {
  if (!out) return LRS_ERR_PARAMETER;
  *out = g_io_err;
  return LRS_OK;
}

}  // extern "C"

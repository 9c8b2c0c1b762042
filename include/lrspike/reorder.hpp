// Matrix Market ingestion and the reorder pipeline:
// read / write Matrix Market coordinate files, strip disconnected rows, symmetric diagonal
// scaling, reverse Cuthill-McKee ordering and permutation.  Host-side structural work (the
// preprocessing that lets real SuiteSparse inputs reach the banded GPU solver).
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "lrspike/matrix.hpp"

namespace lrspike {

/// SPEC.md:39-47.  Coordinate format, real / integer / pattern field, general / symmetric /
/// skew-symmetric; symmetric storage expanded, entries sorted, duplicates summed, 1-based
/// indices made 0-based.  ParseError(line) on malformed input, UnsupportedFieldError on a
/// complex (or hermitian) field or array format.
CsrMatrix read_matrix_market(const std::string& path);
/// General coordinate real, full precision (read -> write -> read is bit-exact).
void write_matrix_market(const std::string& path, const CsrMatrix& a);

/// forward[old] = new, inverse[new] = old.
struct Permutation {
  std::vector<index_t> forward, inverse;
  static Permutation identity(index_t n);
  static Permutation from_order(const std::vector<index_t>& order);  // order[new] = old
};

/// rows / columns whose only entry is the diagonal (or empty) removed;
/// returns the matrix on the retained indices and the removed original indices.
std::pair<CsrMatrix, std::vector<index_t>> strip_disconnected(const CsrMatrix& a);
/// D A D with D = diag(|a_ii|^-1/2); SingularScalingError(row) on a zero
/// (or missing) diagonal.  Returns (scaled matrix, scale) -- row and column scales are equal.
std::pair<CsrMatrix, std::vector<double>> diagonal_scale(const CsrMatrix& a);
/// reverse Cuthill-McKee on the pattern of A + A^T; per connected component
/// (in order of their lowest vertex) the start is a pseudo-peripheral vertex (George-Liu
/// search from the lowest vertex, last-level minimum degree, ties to the lower index);
/// neighbours are visited by ascending (degree, index).
Permutation rcm_ordering(const CsrMatrix& a);
/// B[rowp.forward[i], colp.forward[j]] = A[i, j], rows re-sorted.
CsrMatrix apply_permutation(const CsrMatrix& a, const Permutation& rowp, const Permutation& colp);

}  // namespace lrspike

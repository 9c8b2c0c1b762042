/* Deterministic generators for the BASELINE.json configurations.
 *
 * These are the single source of inputs: the CPU oracle (oracle/) and the
 * CUDA path consume the same bytes.  The reference ships no generator and no
 * test matrices (the paper's SuiteSparse and
 * NESSIE matrices are absent), so the gaps BASELINE.json leaves open are
 * fixed here once and documented in DESIGN.md.
 *
 * All matrices are CSR with int64 indices, strictly increasing columns per
 * row and no duplicates (the CsrMatrix invariants of
 * reference proj/core/include/lrspike/matrix.hpp:17-21).
 */
#ifndef LRS_GEN_H
#define LRS_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lrs_gen_csr {
  int64_t n;
  int64_t nnz;
  int64_t* row_ptr; /* n + 1 */
  int64_t* col_idx; /* nnz */
  double* values;   /* nnz */
} lrs_gen_csr;

/* c1: 2D 5-point Laplacian on a g x g grid, natural ordering idx = y*g + x,
 * diagonal 4 + shift, neighbours -1 (Dirichlet: out-of-grid neighbours are
 * dropped).  Half-bandwidth g. */
int lrs_gen_poisson2d(int64_t g, double shift, lrs_gen_csr* out);

/* c2: 3D 7-point Laplacian on g^3, idx = (z*g + y)*g + x, diagonal 6,
 * neighbours -1, plus a central-difference convection term c*du/dx scaled by
 * h^2 (h = 1/(g+1)): the x+1 neighbour gets +beta and the x-1 neighbour
 * -beta with beta = c*h/2.  Half-bandwidth g^2. */
int lrs_gen_convdiff3d(int64_t g, double conv, lrs_gen_csr* out);

/* c3: 3D 27-point stencil on g^3 with per-cell coefficients
 * kappa = 10^U[-range, range] (seed, LRS_STREAM_MATRIX, ctr = cell).
 * Off-diagonal (p,q) = -2 kp kq / (kp + kq) for all 26 neighbours; diagonal =
 * sum |off| + kappa_p * (number of out-of-grid neighbours) (Dirichlet).
 * Half-bandwidth g^2 + g + 1. */
int lrs_gen_hetero27(int64_t g, uint64_t seed, double log10_range, lrs_gen_csr* out);

/* c4: random banded matrix, n rows, half-bandwidth b, m distinct off-diagonal
 * columns per row sampled without replacement uniformly from
 * [max(0,i-b), min(n-1,i+b)] \ {i}; values N(0,1); diagonal = dom * sum |off|.
 * Rows with fewer than m candidates take all candidates. */
int lrs_gen_randband(int64_t n, int64_t b, int64_t m, uint64_t seed, double dom,
                     lrs_gen_csr* out);

/* c5 base operator A (real): 3D 7-point Laplacian on g^3 (diag 6, off -1) plus
 * a symmetric random perturbation: for each row i one partner j drawn
 * uniformly from [max(0,i-pb), min(n-1,i+pb)] \ {i}, value v ~ N(0, sigma^2)
 * added at (i,j) and (j,i) (duplicates summed).  The solver forms z I - A. */
int lrs_gen_feast_base(int64_t g, uint64_t seed, int64_t pb, double sigma, lrs_gen_csr* out);

void lrs_gen_free(lrs_gen_csr* m);

/* Vectors: kind 0 = uniform[-1,1), 1 = N(0,1), 2 = all ones.  Stream
 * LRS_STREAM_RHS, draw index = element index (column-major for blocks). */
void lrs_gen_vector(int kind, uint64_t seed, int64_t count, double* out);

/* Gaussian test block Omega (rows x cols, column-major) of the randomized
 * spike SVD for (seed, partition, side) -- SPEC.md:289, :312-314. */
void lrs_gen_omega(uint64_t seed, int64_t partition, int side, int64_t rows, int64_t cols,
                   double* out);

#ifdef __cplusplus
}
#endif

#endif /* LRS_GEN_H */

// Tests of the C++ drop-in API (include/lrspike), driven by tests/test_cpp_api.py.
//   test_api cpu   structural host logic (no GPU needed)
//   test_api gpu   factorize / apply / solve through liblrspike_cuda.so
// A tiny check macro stands in for doctest (absent from the image).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "lrspike/errors.hpp"
#include "lrspike/matrix.hpp"
#include "lrspike/solver.hpp"

using namespace lrspike;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                           \
  do {                                                                        \
    if (cond) {                                                               \
      ++g_pass;                                                               \
    } else {                                                                  \
      ++g_fail;                                                               \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
    }                                                                         \
  } while (0)

template <class E>
static bool throws(const std::function<void()>& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static CsrMatrix laplace2d(index_t g, double shift) {
  std::vector<index_t> r, c;
  std::vector<double> v;
  for (index_t y = 0; y < g; ++y)
    for (index_t x = 0; x < g; ++x) {
      const index_t i = y * g + x;
      auto add = [&](index_t j, double a) { r.push_back(i); c.push_back(j); v.push_back(a); };
      add(i, 4.0 + shift);
      if (x > 0) add(i - 1, -1.0);
      if (x < g - 1) add(i + 1, -1.0);
      if (y > 0) add(i - g, -1.0);
      if (y < g - 1) add(i + g, -1.0);
    }
  return CsrMatrix::from_triplets(g * g, g * g, r, c, v);
}

static void cpu_tests() {
  // from_triplets sums duplicates in every row (reference matrix.cpp:96-97 only did row 0)
  {
    auto m = CsrMatrix::from_triplets(3, 3, {0, 1, 1, 2, 1}, {0, 1, 1, 2, 0}, {1, 2, 3, 4, 5});
    CHECK(m.nnz() == 4);
    CHECK(m.coeff(1, 1) == 5.0);
    CHECK(m.coeff(1, 0) == 5.0);
    CHECK(m.coeff(0, 2) == 0.0);
  }
  // validate() errors (matrix.cpp:21-37)
  {
    CsrMatrix m = CsrMatrix::identity(3);
    m.col_idx[1] = 5;
    CHECK(throws<DimensionError>([&] { m.validate(); }));
    CsrMatrix u = CsrMatrix::identity(2);
    u.row_ptr[0] = 1;
    CHECK(throws<DimensionError>([&] { u.validate(); }));
  }
  // band_metrics examples
  {
    auto t = CsrMatrix::from_triplets(4, 4, {0, 0, 1, 1, 1, 2, 2, 2, 3, 3},
                                      {0, 1, 0, 1, 2, 1, 2, 3, 2, 3}, std::vector<double>(10, 1.0));
    auto b = band_metrics(t);
    CHECK(b.band.upper_half_bw == 1 && b.band.lower_half_bw == 1 && b.band.k == 1);
    CHECK(std::fabs(b.band_density - 10.0 / 12.0) < 1e-15);
    auto i = band_metrics(CsrMatrix::identity(5));
    CHECK(i.band.k == 0 && i.diag_weight == 1.0 && i.band_density == 1.0);
  }
  // make_layout
  {
    auto l = make_layout(10, 3, 2);
    CHECK(l.sizes == (std::vector<index_t>{4, 3, 3}));
    CHECK(l.offsets == (std::vector<index_t>{0, 4, 7}));
    CHECK(throws<LayoutError>([] { make_layout(6, 3, 2); }));
    auto s = make_layout(1638, 3, 154);
    CHECK(s.sizes == (std::vector<index_t>{546, 546, 546}));
  }
  // transposed
  {
    auto m = CsrMatrix::from_triplets(2, 3, {0, 1, 1}, {2, 0, 1}, {1, 2, 3});
    auto t = m.transposed();
    CHECK(t.n_rows == 3 && t.coeff(2, 0) == 1.0 && t.coeff(0, 1) == 2.0 && t.coeff(1, 1) == 3.0);
  }
  // extract_blocks: tridiagonal, p = 2, k = 1 -> B_0, C_1 are the
  // boundary scalars; block diagonal -> zero couplings; reassembly is exact
  {
    std::vector<index_t> r, c;
    std::vector<double> v;
    for (index_t i = 0; i < 6; ++i) {
      r.push_back(i); c.push_back(i); v.push_back(4.0 + i);
      if (i + 1 < 6) { r.push_back(i); c.push_back(i + 1); v.push_back(-1.0 - i); }
      if (i > 0) { r.push_back(i); c.push_back(i - 1); v.push_back(-2.0 - i); }
    }
    auto T = CsrMatrix::from_triplets(6, 6, r, c, v);
    auto bl = extract_blocks(T, make_layout(6, 2, 1));
    CHECK(bl.A.size() == 2 && bl.A[0].n_rows == 3 && bl.A[1].coeff(0, 0) == 7.0);
    CHECK(bl.B[0].n_rows == 1 && bl.B[0].coeff(0, 0) == T.coeff(2, 3));
    CHECK(bl.C[1].n_rows == 1 && bl.C[1].coeff(0, 0) == T.coeff(3, 2));
    CHECK(bl.C[0].n_rows == 0 && bl.B[1].n_rows == 0);
    double mism = 0.0;
    for (index_t i = 0; i < 6; ++i)
      for (index_t j = 0; j < 6; ++j) {
        const index_t pi = i / 3, pj = j / 3;
        double e = 0.0;
        if (pi == pj) e = bl.A[pi].coeff(i % 3, j % 3);
        else if (pj == pi + 1 && i == 2 && j == 3) e = bl.B[pi].coeff(0, 0);
        else if (pi == pj + 1 && i == 3 && j == 2) e = bl.C[pi].coeff(0, 0);
        mism += std::fabs(e - T.coeff(i, j));
      }
    CHECK(mism == 0.0);
    auto D = CsrMatrix::from_triplets(4, 4, {0, 1, 2, 3}, {0, 1, 2, 3}, {1, 2, 3, 4});
    auto bd = extract_blocks(D, make_layout(4, 2, 1));
    CHECK(bd.B[0].nnz() == 0 && bd.C[1].nnz() == 0);
    bool got = false;
    try {
      extract_blocks(T, make_layout(6, 3, 0));
    } catch (const NotBlockTridiagonalError& e) {
      got = e.row() == 1 && e.col() == 2;
    }
    CHECK(got);
  }
}

static double resid(const CsrMatrix& a, const DenseBlock& x, const DenseBlock& b) {
  double rn = 0, bn = 0;
  for (index_t i = 0; i < a.n_rows; ++i) {
    double s = 0;
    for (index_t p = a.row_ptr[i]; p < a.row_ptr[i + 1]; ++p) s += a.values[p] * x(a.col_idx[p], 0);
    rn += (b(i, 0) - s) * (b(i, 0) - s);
    bn += b(i, 0) * b(i, 0);
  }
  return std::sqrt(rn / bn);
}

static void gpu_tests() {
  // identity: spmv, solve_block, BiCGStab converges at 0.5 iterations
  {
    auto I = CsrMatrix::identity(300);
    DenseBlock b(300, 1);
    for (index_t i = 0; i < 300; ++i) b(i, 0) = std::sin(0.1 * i) + 1.0;
    auto y = spmv(I, b);
    CHECK(y(17, 0) == b(17, 0));
    SolverConfig cfg;
    cfg.p = 2;
    cfg.k = 1;
    cfg.n_svd = 0;
    auto r = solve(I, b, cfg);
    CHECK(r.second.converged);
    CHECK(r.second.iterations == 0.5);
    CHECK(std::fabs(r.first(5, 0) - b(5, 0)) < 1e-14);
  }
  // factorize_block / solve_block: identity, diag(2, 4), adjoint
  {
    auto fb = factorize_block(CsrMatrix::identity(5));
    DenseBlock b(5, 2);
    for (index_t i = 0; i < 5; ++i) b(i, 0) = i + 1.0, b(i, 1) = -2.0 * i;
    auto x = solve_block(fb, b);
    CHECK(fb.n() == 5 && x(3, 0) == 4.0 && x(4, 1) == -8.0);
    auto fd = factorize_block(CsrMatrix::from_triplets(2, 2, {0, 1}, {0, 1}, {2.0, 4.0}));
    DenseBlock q(2, 1);
    q(0, 0) = 4.0;
    q(1, 0) = 4.0;
    auto xd = solve_block(fd, q);
    CHECK(xd(0, 0) == 2.0 && xd(1, 0) == 1.0);
    auto fu = factorize_block(CsrMatrix::from_triplets(2, 2, {0, 0, 1}, {0, 1, 1}, {1.0, 2.0, 1.0}));
    DenseBlock e1(2, 1);
    e1(0, 0) = 1.0;
    auto xa = solve_block_adjoint(fu, e1);
    CHECK(xa(0, 0) == 1.0 && xa(1, 0) == -2.0);
  }
  // adjoint solve of [[1,2],[0,1]]: e1 -> (1,-2), one 2x2 block (p=1)
  {
    auto m = CsrMatrix::from_triplets(2, 2, {0, 0, 1}, {0, 1, 1}, {1.0, 2.0, 1.0});
    SolverConfig cfg;
    cfg.p = 1;
    cfg.k = 1;
    cfg.n_svd = 0;
    cfg.variant = Variant::BLOCK_JACOBI;
    auto f = factorize(m, cfg);
    DenseBlock e1(2, 1);
    e1(0, 0) = 1.0;
    auto x = f->solve_block_adjoint(0, e1);
    CHECK(std::fabs(x(0, 0) - 1.0) < 1e-15 && std::fabs(x(1, 0) + 2.0) < 1e-15);
  }
  // 2D Laplacian 40x40, p=4: LR-SPIKE-T + GMRES and BiCGStab converge; n_svd=0 == Block Jacobi
  {
    auto A = laplace2d(40, 1e-2);
    DenseBlock b(A.n_rows, 1);
    for (index_t i = 0; i < A.n_rows; ++i) b(i, 0) = std::cos(0.37 * i);
    SolverConfig cfg;
    cfg.p = 4;
    cfg.k = 40;
    cfg.n_svd = 8;
    cfg.outer.method = Method::GMRES;
    cfg.outer.restart = 30;
    auto f = factorize(A, cfg);
    CHECK(f->n_svd() == 8);
    auto g = solve(A, b, cfg, f);
    CHECK(g.second.converged);
    CHECK(resid(A, g.first, b) <= 1e-8);
    cfg.outer.method = Method::BICGSTAB;
    auto bi = solve(A, b, cfg, f);
    CHECK(bi.second.converged);
    CHECK(resid(A, bi.first, b) <= 1e-8);
    // ledger exactness: 4 (p-1) n_svd n_rhs scalars per application
    CHECK(bi.second.ledger.precond_apply.scalars + bi.second.ledger.recovery.scalars ==
          4 * 3 * 8 * bi.second.precond_applications);
    SolverConfig c0 = cfg;
    c0.n_svd = 0;
    auto f0 = factorize(A, c0);
    auto x1 = apply_precond_T(*f0, b), x2 = apply_block_jacobi(*f0, b);
    bool same = true;
    for (index_t i = 0; i < A.n_rows; ++i) same &= x1(i, 0) == x2(i, 0);
    CHECK(same);
    // LR-SPIKE-I (inner reduced BiCGStab) and LR-SPIKE-OTF (exact reduced system)
    SolverConfig ci = cfg;
    ci.variant = Variant::LR_SPIKE_I;
    auto fi = factorize(A, ci);
    auto xi = apply_precond_I(*fi, b);
    CHECK(xi.rows() == A.n_rows);
    auto si = solve(A, b, ci, fi);
    CHECK(si.second.converged && resid(A, si.first, b) <= 1e-8);
    CHECK(si.second.inner_solves == si.second.precond_applications);
    CHECK(si.second.inner_iterations > 0);
    CHECK(throws<ParameterError>([&] { apply_precond_I(*f, b); }));
    SolverConfig co = cfg;
    co.variant = Variant::LR_SPIKE_OTF;
    auto so = solve(A, b, co);
    CHECK(so.second.converged && resid(A, so.first, b) <= 1e-8);
    CHECK(so.second.ledger.reduced_matvec.scalars % (2 * 3 * 40) == 0);
    // CG with the (symmetric) Block Jacobi preconditioner on the SPD Laplacian
    SolverConfig cg = cfg;
    cg.variant = Variant::BLOCK_JACOBI;
    cg.n_svd = 0;
    cg.outer.method = Method::CG;
    auto sc = solve(A, b, cg);
    CHECK(sc.second.converged && resid(A, sc.first, b) <= 1e-8);
    // errors: layout infeasible, not block tridiagonal
    SolverConfig bad = cfg;
    bad.p = 400;
    CHECK(throws<LayoutError>([&] { factorize(A, bad); }));
    SolverConfig nbt = cfg;
    nbt.k = 10;
    bool got = false;
    try {
      factorize(A, nbt);
    } catch (const NotBlockTridiagonalError& e) {
      got = e.row() >= 0 && e.col() >= 0;
    } catch (...) {
    }
    CHECK(got);
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_tests();
  if (mode == "gpu") gpu_tests();
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}

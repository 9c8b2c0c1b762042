// Tests of the C++ drop-in API (include/lrspike), driven by tests/test_cpp_api.py.
//   test_api cpu   structural host logic (no GPU needed)
//   test_api gpu   factorize / apply / solve through liblrspike_cuda.so
// A tiny check macro stands in for doctest (absent from the image).
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "lrspike/comm.hpp"
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

// ---- oracle fixtures (written by tests/test_gpu_cpp_api.py from the CPU oracle) ----------
// manifest.txt: "<name> <rows> <cols> <f64|c128|i64> <extra int>" per line; <name>.bin raw
struct Fixtures {
  std::string dir;
  std::map<std::string, std::vector<long>> meta;
  explicit Fixtures(const std::string& d) : dir(d) {
    std::ifstream m(d + "/manifest.txt");
    std::string line;
    while (std::getline(m, line)) {
      std::istringstream is(line);
      std::string name, type;
      long r, c, extra = 0;
      is >> name >> r >> c >> type >> extra;
      meta[name] = {r, c, type == "f64" ? 1L : type == "c128" ? 2L : 3L, extra};
    }
  }
  long rows(const std::string& n) const { return meta.at(n)[0]; }
  long cols(const std::string& n) const { return meta.at(n)[1]; }
  long extra(const std::string& n) const { return meta.at(n)[3]; }
  template <class T>
  std::vector<T> raw(const std::string& n) const {
    std::ifstream f(dir + "/" + n + ".bin", std::ios::binary);
    f.seekg(0, std::ios::end);
    const size_t bytes = (size_t)f.tellg();
    f.seekg(0);
    std::vector<T> v(bytes / sizeof(T));
    f.read(reinterpret_cast<char*>(v.data()), (std::streamsize)bytes);
    return v;
  }
  template <class S>
  DenseBlockT<S> block(const std::string& n) const {
    DenseBlockT<S> b(rows(n), cols(n));
    const auto v = raw<S>(n);
    std::copy(v.begin(), v.end(), b.data());
    return b;
  }
  template <class S>
  CsrMatrixT<S> csr(const std::string& n) const {
    CsrMatrixT<S> a;
    a.n_rows = a.n_cols = rows(n + "_rowptr") - 1;
    a.row_ptr = raw<index_t>(n + "_rowptr");
    a.col_idx = raw<index_t>(n + "_colidx");
    a.values = raw<S>(n + "_values");
    return a;
  }
};

template <class S>
static double rel(const DenseBlockT<S>& a, const DenseBlockT<S>& b) {
  double d = 0, n = 0;
  for (index_t e = 0; e < a.size(); ++e) {
    d += std::norm(a.data()[e] - b.data()[e]);
    n += std::norm(b.data()[e]);
  }
  return std::sqrt(d / std::max(n, 1e-300));
}

template <class S>
static DenseBlockT<S> usv(const LowRankSpikeT<S>& s) {  // u diag(sigma) v
  DenseBlockT<S> o(s.u.rows(), s.v.cols());
  for (index_t a = 0; a < (index_t)s.sigma.size(); ++a)
    for (index_t j = 0; j < s.v.cols(); ++j) {
      const S w = s.sigma[a] * s.v(a, j);
      for (index_t i = 0; i < s.u.rows(); ++i) o(i, j) += s.u(i, a) * w;
    }
  return o;
}

static void report(const char* what, double v, double bar) {
  std::printf("  %-44s %.3e (bar %.0e)\n", what, v, bar);
  CHECK(v <= bar);
}

static void oracle_tests(const std::string& dir) {
  Fixtures F(dir);
  // ---- real case (c1 structure): every SPEC op of the C++ surface against the oracle
  {
    const auto A = F.csr<double>("A");
    const index_t p = F.extra("A_rowptr"), k = F.extra("A_colidx"), r = F.extra("A_values");
    const auto lay = make_layout(A.n_rows, p, k);
    const auto blocks = extract_blocks(A, lay);
    // randomized_spike_svd, both sides, and the coupling mode
    const auto F0 = factorize_block(blocks.A[0]);
    const auto F1 = factorize_block(blocks.A[1]);
    const index_t os = (r + 1) / 2;
    const auto sT = randomized_spike_svd(F0, blocks.B[0], Side::T, r, os, 2, F.extra("rhs"), 0);
    const auto sW = randomized_spike_svd(F1, blocks.C[1], Side::W, r, os, 2, F.extra("rhs"), 1);
    const auto sC = randomized_spike_svd(F0, blocks.B[0], Side::T, r, os, 2, F.extra("rhs"), 0,
                                         SpikeMode::CouplingSvd);
    report("randomized_spike_svd T_0: u S v", rel(usv(sT), F.block<double>("usvT0")), 1e-9);
    report("randomized_spike_svd W_1: u S v", rel(usv(sW), F.block<double>("usvW1")), 1e-9);
    report("coupling-mode spike T_0: u S v", rel(usv(sC), F.block<double>("usvC0")), 1e-9);
    DenseBlock sig(r, 1);
    for (index_t a = 0; a < r; ++a) sig(a, 0) = sT.sigma[a];
    report("randomized_spike_svd T_0: sigma", rel(sig, F.block<double>("sigT0")), 1e-10);
    const auto tips = spike_tips(sT, k);
    CHECK(tips.first.rows() == k && tips.second.rows() == k && tips.second(0, 0) == sT.u(sT.u.rows() - k, 0));
    // build / apply_truncated_precond and matvec_lowrank from the ORACLE's spikes
    std::vector<LowRankSpike> spT, spW;
    for (index_t i = 0; i + 1 < p; ++i) {
      LowRankSpike t, w;
      t.u = F.block<double>("uT" + std::to_string(i));
      t.v = F.block<double>("vT" + std::to_string(i));
      w.u = F.block<double>("uW" + std::to_string(i + 1));
      w.v = F.block<double>("vW" + std::to_string(i + 1));
      const auto st = F.block<double>("sT" + std::to_string(i));
      const auto sw = F.block<double>("sW" + std::to_string(i + 1));
      t.sigma.assign(st.data(), st.data() + st.size());
      w.sigma.assign(sw.data(), sw.data() + sw.size());
      w.side = Side::W;
      spT.push_back(t);
      spW.push_back(w);
    }
    const auto P = build_truncated_precond(spT, spW, k);
    ReducedVector g(p, k, 2);
    g.data = F.block<double>("g");
    report("apply_truncated_precond", rel(apply_truncated_precond(*P, g).data, F.block<double>("trunc_g")), 1e-12);
    report("matvec_lowrank", rel(matvec_lowrank(*P, g).data, F.block<double>("lowrank_g")), 1e-12);
    // Krylov drivers on operator contracts: A = SpMV, M = LR-SPIKE-T
    SolverConfig cfg;
    cfg.p = p;
    cfg.k = k;
    cfg.n_svd = r;
    cfg.seed = F.extra("rhs");
    auto fac = factorize(A, cfg);
    const auto b = F.block<double>("rhs");
    const auto opA = as_operator(*fac->matrix());
    const auto opM = as_operator(*fac);
    IterConfig it;
    it.tol = 1e-8;
    auto bi = bicgstab(opA, &opM, b, it);
    report("bicgstab(operators) x vs oracle", rel(bi.first, F.block<double>("x_bicgstab")), 1e-8);
    CHECK(std::fabs(bi.second.iterations - F.extra("x_bicgstab")) <= 2 && bi.second.residual_final <= 1e-8);
    it.restart = 30;
    auto gm = gmres(opA, &opM, b, it);
    report("gmres(operators) x vs oracle", rel(gm.first, F.block<double>("x_gmres")), 1e-8);
    CHECK(std::fabs(gm.second.iterations - F.extra("x_gmres")) <= 2 && gm.second.residual_final <= 1e-8);
    // matvec_exact / matvec_otf on the factorization vs the oracle's exact reduced matvec
    report("matvec_exact (otf)", rel(matvec_exact(*fac, g).data, F.block<double>("exact_g")), 1e-11);
    // spmv reuses the device copy: same result, no re-upload
    const auto y1 = spmv(A, b);
    const auto y2 = spmv(A, b);
    CHECK(A.device_cache && rel(y1, y2) == 0.0);
    // factorize_dist on a one-rank in-library NCCL communicator == factorize
    try {
      NcclCommunicator comm(Device::default_device(), NcclCommunicator::nccl_unique_id(), 0, 1);
      auto fd = factorize_dist(A, cfg, comm);
      const auto xd = solve(A, b, cfg, fd);
      const auto xs = solve(A, b, cfg, fac);
      report("factorize_dist (1-rank NCCL) vs factorize", rel(xd.first, xs.first), 0.0);
    } catch (const Error& e) {
      std::printf("  NCCL communicator unavailable: %s\n", e.what());
      CHECK(false);
    }
  }
  // ---- complex128 (c5 structure, 2 RHS): solve through the templated API
  {
    const auto Az = F.csr<complex128>("Z");
    SolverConfigZ cz;
    cz.p = F.extra("Z_rowptr");
    cz.k = F.extra("Z_colidx");
    cz.n_svd = F.extra("Z_values");
    cz.seed = F.extra("zrhs");
    cz.outer.method = Method::GMRES;
    cz.outer.restart = 40;
    cz.outer.tol = 1e-10;
    const auto bz = F.block<complex128>("zrhs");
    const auto sz = solve(Az, bz, cz);
    report("complex128 GMRES solve x vs oracle", rel(sz.first, F.block<complex128>("zx")), 1e-8);
    CHECK(sz.second.converged && sz.second.residual_final <= 1e-10);
    CHECK(std::fabs(sz.second.iterations - F.extra("zx")) <= 2);
    const auto fz = factorize(Az, cz);
    const auto spz = fz->spike(0, Side::T);
    report("complex128 spike T_0: u S v", rel(usv(spz), F.block<complex128>("zusvT0")), 1e-9);
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_tests();
  if (mode == "gpu") gpu_tests();
  if (mode == "oracle" && argc > 2) oracle_tests(argv[2]);
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}

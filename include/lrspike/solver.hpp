// lrspike partition / spike_solvers / krylov operations of the C++ drop-in API.
//
// Names follow the SPEC operations: make_layout, factorize,
// solve_block, solve_block_adjoint, apply_precond_T, apply_block_jacobi, solve,
// with SolverConfig / IterConfig / SolveReport / CommLedger.  GMRES(m) is added
// as Method::GMRES.  Everything executes on the GPU through the
// C-ABI (include/lrspike_capi.h); the classes here only own handles.
#pragma once

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "lrspike/errors.hpp"
#include "lrspike/matrix.hpp"

struct lrs_ctx;
struct lrs_mat;
struct lrs_fact;

namespace lrspike {

/// SPEC.md:157-162.
struct PartitionLayout {
  index_t p = 1;
  std::vector<index_t> sizes;
  std::vector<index_t> offsets;
  index_t k = 0;
};

/// first (n mod p) partitions get ceil(n/p) rows; every n_i > k.
PartitionLayout make_layout(index_t n, index_t p, index_t k);

// Table 1 of the paper / SPEC.md:470
enum class Variant { LR_SPIKE_T, BLOCK_JACOBI, LR_SPIKE_I, LR_SPIKE_OTF };
enum class Method { BICGSTAB, GMRES, CG };  // CG: SPEC.md:430-436

/// SPEC.md:411-414 (+ method / restart).
struct IterConfig {
  double tol = 1e-8;
  index_t max_iters = 1000;
  double breakdown_eps = 1e-30;
  const DenseBlock* initial_guess = nullptr;
  Method method = Method::BICGSTAB;
  int restart = 30;
};

/// SPEC.md:470-473.
enum class SpikeMode { SpikeSvd, CouplingSvd };

struct SolverConfig {
  Variant variant = Variant::LR_SPIKE_T;
  index_t p = 4;
  index_t k = 0;  // 0 -> band_metrics(A).band.k
  index_t n_svd = 8;
  index_t oversample = -1;  // -1 -> ceil(n_svd / 2)
  int passes = 2;
  std::uint64_t seed = 0;
  IterConfig outer;
  // LR-SPIKE-I inner reduced solve (BiCGStab); LR-SPIKE-OTF reduced solve
  double inner_tol = 1e-12;
  index_t inner_max_iters = 200;
  double otf_tol = 1e-8;
  index_t otf_max_iters = 500;
  int otf_escalations = 4;
  // FP32 off-diagonal factor tiles in the preconditioner applies
  bool factor_fp32 = false;
  // how the low-rank spikes are built: the SPEC's randomized spike SVD, or
  // the truncated SVD of B_i / C_i followed by padded solves (north_star setup (1))
  SpikeMode spike_mode = SpikeMode::SpikeSvd;
};

/// SPEC.md:466-469.
struct CommLedger {
  struct Stage {
    index_t messages = 0;
    index_t scalars = 0;
  };
  Stage reduced_matvec, precond_apply, recovery;
};

/// SPEC.md:415-419.
struct SolveReport {
  bool converged = false;
  double iterations = 0.0;
  std::vector<double> residual_history;
  index_t precond_applications = 0;
  index_t matvecs = 0;
  index_t comm_scalars = 0;
  CommLedger ledger;
  std::uint64_t seed = 0;
  double wall_time = 0.0;
  double residual_final = 0.0;
  double inner_iterations = 0.0;  // LR-SPIKE-I: inner half-iterations summed over applies
  index_t inner_solves = 0;
};

/// A CUDA device + stream (lrs_ctx).  device() returns the process default (GPU 0).
class Device {
 public:
  explicit Device(int ordinal = 0);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  lrs_ctx* handle() const { return h_; }
  static Device& default_device();

 private:
  lrs_ctx* h_ = nullptr;
};

/// A CsrMatrix resident on the device (lrs_mat).
class DeviceMatrix {
 public:
  DeviceMatrix(const CsrMatrix& a, Device& dev = Device::default_device());
  ~DeviceMatrix();
  DeviceMatrix(const DeviceMatrix&) = delete;
  DeviceMatrix& operator=(const DeviceMatrix&) = delete;
  lrs_mat* handle() const { return h_; }
  index_t n() const { return n_; }
  Device& device() const { return *dev_; }
  DenseBlock spmv(const DenseBlock& x) const;

 private:
  lrs_mat* h_ = nullptr;
  index_t n_ = 0;
  Device* dev_;
};

/// layout, block factors, low-rank spikes, truncated preconditioner.
/// Immutable after construction and reusable across solves.
class SpikeFactorization {
 public:
  SpikeFactorization(std::shared_ptr<DeviceMatrix> a, const SolverConfig& cfg);
  ~SpikeFactorization();
  SpikeFactorization(const SpikeFactorization&) = delete;
  SpikeFactorization& operator=(const SpikeFactorization&) = delete;

  const PartitionLayout& layout() const { return layout_; }
  index_t n_svd() const { return n_svd_; }
  const SolverConfig& config() const { return cfg_; }
  double factorize_seconds() const { return t_factorize_; }
  CommLedger ledger() const;
  lrs_fact* handle() const { return h_; }
  const std::shared_ptr<DeviceMatrix>& matrix() const { return a_; }

  /// SPEC.md:226-234 / :235-241 on partition i.
  DenseBlock solve_block(index_t i, const DenseBlock& rhs) const;
  DenseBlock solve_block_adjoint(index_t i, const DenseBlock& rhs) const;
  /// Low-rank spike (u n_i x r, sigma, v r x k) of partition i, side 0 = T, 1 = W.
  void spike(index_t i, int side, DenseBlock& u, std::vector<double>& sigma, DenseBlock& v) const;

 private:
  std::shared_ptr<DeviceMatrix> a_;
  SolverConfig cfg_;
  lrs_fact* h_ = nullptr;
  PartitionLayout layout_;
  index_t n_svd_ = 0;
  double t_factorize_ = 0.0;
};

/// the diagonal blocks A_i and the k x k corner couplings B_i (bottom-left
/// of the super-diagonal block, coupling partition i to i+1; i = 0..p-2) and C_i (top-right
/// of the sub-diagonal block, coupling i to i-1; i = 1..p-1, C[0] empty).  The couplings are
/// kept sparse.  Throws NotBlockTridiagonalError(row, col) at the first entry
/// (row-major) outside the pattern.  Host-side data movement only.
struct PartitionBlocks {
  PartitionLayout layout;
  std::vector<CsrMatrix> A, B, C;
};
PartitionBlocks extract_blocks(const CsrMatrix& a, const PartitionLayout& layout);

/// SPEC.md:211-225 (BlockFactor / factorize_block): the LU of one block on the GPU (the
/// p = 1 Block Jacobi factorization of A_i).
class BlockFactor {
 public:
  explicit BlockFactor(std::shared_ptr<SpikeFactorization> f) : f_(std::move(f)) {}
  index_t n() const;
  const SpikeFactorization& factorization() const { return *f_; }

 private:
  std::shared_ptr<SpikeFactorization> f_;
};
BlockFactor factorize_block(const CsrMatrix& a_i);
/// SPEC.md:226-234 / :235-241.
DenseBlock solve_block(const BlockFactor& f, const DenseBlock& rhs);
DenseBlock solve_block_adjoint(const BlockFactor& f, const DenseBlock& rhs);

/// SPEC.md:476-484.
std::shared_ptr<SpikeFactorization> factorize(const CsrMatrix& a, const SolverConfig& cfg);
/// SPEC.md:485-493.
DenseBlock apply_precond_T(const SpikeFactorization& f, const DenseBlock& rhs);
/// SPEC.md:494-502 (an LR_SPIKE_I factorization; inner BiCGStab on the reduced system).
DenseBlock apply_precond_I(const SpikeFactorization& f, const DenseBlock& rhs);
/// SPEC.md:512-519.
DenseBlock apply_block_jacobi(const SpikeFactorization& f, const DenseBlock& rhs);
/// factorize (or reuse f) and run the outer Krylov method.
/// Non-convergence is reported (report.converged == false), not thrown.
std::pair<DenseBlock, SolveReport> solve(const CsrMatrix& a, const DenseBlock& rhs,
                                         const SolverConfig& cfg,
                                         std::shared_ptr<SpikeFactorization> f = nullptr);

}  // namespace lrspike

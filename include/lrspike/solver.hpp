// lrspike partition / block_solver / spikes / reduced_system / krylov / spike_solvers
// operations of the C++ drop-in API.
//
// Names follow the SPEC operations: make_layout, extract_blocks, factorize_block,
// solve_block, solve_block_adjoint, randomized_spike_svd, spike_tips,
// build_truncated_precond, apply_truncated_precond, matvec_exact / matvec_lowrank /
// matvec_otf, bicgstab, cg, factorize, apply_precond_T / _I, apply_block_jacobi, solve,
// with SolverConfig / IterConfig / SolveReport / CommLedger.  GMRES(m) is added as
// Method::GMRES and gmres().  Everything is templated on the scalar
// (double, complex128 for config c5); the unsuffixed names are the double
// instances, the Z-suffixed ones complex128.  Every numerical operation executes on the
// GPU through the C-ABI (include/lrspike_capi.h); the classes here only own handles and
// move host blocks.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <utility>
#include <vector>

#include "lrspike/errors.hpp"
#include "lrspike/matrix.hpp"

struct lrs_ctx;
struct lrs_mat;
struct lrs_fact;

namespace lrspike {

class Communicator;  // lrspike/comm.hpp

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
/// How the low-rank spikes are built: the SPEC's randomized SVD of the
/// spike, or the truncated SVD of B_i / C_i followed by padded solves
/// against its singular vectors (BASELINE.json north_star setup (1)).
enum class SpikeMode { SpikeSvd, CouplingSvd };
/// Spike side: T_i = A_i^-1 [0; B_i] (i < p-1), W_i = A_i^-1 [C_i; 0] (i > 0).
enum class Side { T = 0, W = 1 };

/// SPEC.md:411-414 (+ method / GMRES restart).
template <class S>
struct IterConfigT {
  double tol = 1e-8;
  index_t max_iters = 1000;
  double breakdown_eps = 1e-30;
  const DenseBlockT<S>* initial_guess = nullptr;
  Method method = Method::BICGSTAB;
  int restart = 30;
};
using IterConfig = IterConfigT<double>;
using IterConfigZ = IterConfigT<complex128>;

/// SPEC.md:470-473.
template <class S>
struct SolverConfigT {
  Variant variant = Variant::LR_SPIKE_T;
  index_t p = 4;
  index_t k = 0;  // 0 -> band_metrics(A).band.k
  index_t n_svd = 8;
  index_t oversample = -1;  // -1 -> ceil(n_svd / 2)
  int passes = 2;
  std::uint64_t seed = 0;
  IterConfigT<S> outer;
  // LR-SPIKE-I inner reduced solve (BiCGStab); LR-SPIKE-OTF reduced solve
  double inner_tol = 1e-12;
  index_t inner_max_iters = 200;
  double otf_tol = 1e-8;
  index_t otf_max_iters = 500;
  int otf_escalations = 4;
  // FP32 off-diagonal factor tiles in the preconditioner applies
  bool factor_fp32 = false;
  SpikeMode spike_mode = SpikeMode::SpikeSvd;
};
using SolverConfig = SolverConfigT<double>;
using SolverConfigZ = SolverConfigT<complex128>;

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
  bool breakdown = false;
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
  // host round trips: transport calls, stream syncs a host-callback transport forced before
  // them (0 with NcclCommunicator), syncs to read the Krylov scalars
  index_t comm_calls = 0, comm_host_syncs = 0, scalar_syncs = 0;
};

/// A CUDA device + stream (lrs_ctx).  The context outlives its matrices and factorizations
/// (the library defers its teardown until the last of them is destroyed).
class Device {
 public:
  explicit Device(int ordinal = 0);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  lrs_ctx* handle() const { return h_; }
  /// The process default (GPU 0), created on first use.
  static Device& default_device();

 private:
  lrs_ctx* h_ = nullptr;
};

/// Column-major device block handed to operator callbacks: rows x cols, leading dim ld.
template <class S>
struct DeviceView {
  S* data = nullptr;
  index_t rows = 0, cols = 0, ld = 0;
};

/// A CsrMatrix resident on the device (lrs_mat).
template <class S>
class DeviceMatrixT {
 public:
  explicit DeviceMatrixT(const CsrMatrixT<S>& a, Device& dev = Device::default_device());
  ~DeviceMatrixT();
  DeviceMatrixT(const DeviceMatrixT&) = delete;
  DeviceMatrixT& operator=(const DeviceMatrixT&) = delete;
  lrs_mat* handle() const { return h_; }
  index_t n() const { return n_; }
  Device& device() const { return *dev_; }
  /// y = A x (host blocks).
  DenseBlockT<S> spmv(const DenseBlockT<S>& x) const;
  /// y (+)= A x on device blocks (no host copies).
  void spmv_device(DeviceView<const S> x, DeviceView<S> y, bool accumulate = false) const;

 private:
  lrs_mat* h_ = nullptr;
  index_t n_ = 0;
  Device* dev_;
};
using DeviceMatrix = DeviceMatrixT<double>;
using DeviceMatrixZ = DeviceMatrixT<complex128>;

/// T_i ~ u diag(sigma) v with u n_i x r (orthonormal columns), sigma
/// non-increasing, v r x k (orthonormal rows).
template <class S>
struct LowRankSpikeT {
  DenseBlockT<S> u;
  std::vector<double> sigma;
  DenseBlockT<S> v;
  Side side = Side::T;
  bool rank_collapsed = false;  // sigma_j < 1e-14 sigma_1 were truncated
};
using LowRankSpike = LowRankSpikeT<double>;
using LowRankSpikeZ = LowRankSpikeT<complex128>;

/// (top k rows of u, bottom k rows of u).
template <class S>
std::pair<DenseBlockT<S>, DenseBlockT<S>> spike_tips(const LowRankSpikeT<S>& s, index_t k) {
  if (k < 0 || k > s.u.rows()) throw DimensionError("spike_tips: k exceeds the spike height");
  return {s.u.middle_rows(0, k), s.u.middle_rows(s.u.rows() - k, k)};
}

/// layout, block factors, low-rank spikes, truncated preconditioner.
/// Immutable after construction and reusable across solves.  A sharded
/// factorization (factorize_dist) owns a contiguous block of partitions of this rank.
template <class S>
class SpikeFactorizationT {
 public:
  SpikeFactorizationT(std::shared_ptr<DeviceMatrixT<S>> a, const SolverConfigT<S>& cfg,
                      Communicator* comm = nullptr);
  ~SpikeFactorizationT();
  SpikeFactorizationT(const SpikeFactorizationT&) = delete;
  SpikeFactorizationT& operator=(const SpikeFactorizationT&) = delete;

  const PartitionLayout& layout() const { return layout_; }
  index_t n_svd() const { return n_svd_; }
  const SolverConfigT<S>& config() const { return cfg_; }
  double factorize_seconds() const { return t_factorize_; }
  CommLedger ledger() const;
  lrs_fact* handle() const { return h_; }
  const std::shared_ptr<DeviceMatrixT<S>>& matrix() const { return a_; }
  /// Rows [row_lo, row_hi) this rank owns (all rows on one GPU).
  index_t row_lo() const { return row_lo_; }
  index_t row_hi() const { return row_hi_; }

  /// SPEC.md:226-234 / :235-241 on partition i.
  DenseBlockT<S> solve_block(index_t i, const DenseBlockT<S>& rhs) const;
  DenseBlockT<S> solve_block_adjoint(index_t i, const DenseBlockT<S>& rhs) const;
  /// The low-rank spike of partition i (side T: i < p-1, W: i > 0) the factorization built.
  LowRankSpikeT<S> spike(index_t i, Side side) const;
  /// out = M^-1 in on device blocks: the factorization's own preconditioner (T, I, BJ).
  void apply_device(DeviceView<const S> in, DeviceView<S> out) const;

 private:
  std::shared_ptr<DeviceMatrixT<S>> a_;
  SolverConfigT<S> cfg_;
  lrs_fact* h_ = nullptr;
  PartitionLayout layout_;
  index_t n_svd_ = 0, row_lo_ = 0, row_hi_ = 0;
  double t_factorize_ = 0.0;
};
using SpikeFactorization = SpikeFactorizationT<double>;
using SpikeFactorizationZ = SpikeFactorizationT<complex128>;

/// the diagonal blocks A_i and the k x k corner couplings B_i (bottom-left
/// of the super-diagonal block, coupling partition i to i+1; i = 0..p-2) and C_i (top-right
/// of the sub-diagonal block, coupling i to i-1; i = 1..p-1, C[0] empty).  The couplings are
/// kept sparse.  Throws NotBlockTridiagonalError(row, col) at the first entry
/// (row-major) outside the pattern.  Host-side data movement only.
template <class S>
struct PartitionBlocksT {
  PartitionLayout layout;
  std::vector<CsrMatrixT<S>> A, B, C;
};
using PartitionBlocks = PartitionBlocksT<double>;
template <class S>
PartitionBlocksT<S> extract_blocks(const CsrMatrixT<S>& a, const PartitionLayout& layout);

/// SPEC.md:211-225 (BlockFactor / factorize_block): the banded LU of one block on the GPU
/// (the p = 1 Block Jacobi factorization of A_i).
template <class S>
class BlockFactorT {
 public:
  explicit BlockFactorT(std::shared_ptr<SpikeFactorizationT<S>> f) : f_(std::move(f)) {}
  index_t n() const { return f_->layout().sizes.at(0); }
  const SpikeFactorizationT<S>& factorization() const { return *f_; }

 private:
  std::shared_ptr<SpikeFactorizationT<S>> f_;
};
using BlockFactor = BlockFactorT<double>;
template <class S>
BlockFactorT<S> factorize_block(const CsrMatrixT<S>& a_i, Device& dev = Device::default_device());
/// SPEC.md:226-234 / :235-241.
template <class S>
DenseBlockT<S> solve_block(const BlockFactorT<S>& f, const DenseBlockT<S>& rhs);
template <class S>
DenseBlockT<S> solve_block_adjoint(const BlockFactorT<S>& f, const DenseBlockT<S>& rhs);

/// rank-n_svd randomized SVD of the spike of block F with the k x k
/// coupling (B_i for side T, C_i for side W): Omega ~ N(0,1)^{k x l} from the stream
/// (seed, partition, side), Y = F^-1 pad(coupling Omega), Q = orth(Y),
/// (passes - 2) / 2 power passes, Z^H = coupling^H (F^-H Q)|tip, SVD(Z).  mode =
/// CouplingSvd builds the spike from the truncated SVD of the coupling instead.  Every
/// step runs on the GPU (band solves, SpMV, QR, Jacobi SVD, small GEMMs).
template <class S>
LowRankSpikeT<S> randomized_spike_svd(const BlockFactorT<S>& F, const CsrMatrixT<S>& coupling,
                                      Side side, index_t n_svd, index_t oversample, int passes,
                                      std::uint64_t seed, index_t partition,
                                      SpikeMode mode = SpikeMode::SpikeSvd);

/// the tips of a reduced vector, stored as one 2kp x n_rhs block
/// (partition i's top tip in rows [2ki, 2ki + k), its bottom tip in [2ki + k, 2k(i+1))).
template <class S>
struct ReducedVectorT {
  index_t p = 0, k = 0;
  DenseBlockT<S> data;
  ReducedVectorT() = default;
  ReducedVectorT(index_t p_, index_t k_, index_t n_rhs) : p(p_), k(k_), data(2 * k_ * p_, n_rhs) {}
  DenseBlockT<S> top(index_t i) const { return data.middle_rows(2 * k * i, k); }
  DenseBlockT<S> bottom(index_t i) const { return data.middle_rows(2 * k * i + k, k); }
};
using ReducedVector = ReducedVectorT<double>;

/// the truncated preconditioner (per interface G = K^-1 and the LU of H)
/// on the device, built from explicit spikes.
template <class S>
class TruncatedPrecondT {
 public:
  TruncatedPrecondT(lrs_fact* h, Device& dev, index_t p, index_t k, index_t r)
      : h_(h), dev_(&dev), p_(p), k_(k), r_(r) {}
  ~TruncatedPrecondT();
  TruncatedPrecondT(const TruncatedPrecondT&) = delete;
  TruncatedPrecondT& operator=(const TruncatedPrecondT&) = delete;
  lrs_fact* handle() const { return h_; }
  Device& device() const { return *dev_; }
  index_t p() const { return p_; }
  index_t k() const { return k_; }
  index_t n_svd() const { return r_; }

 private:
  lrs_fact* h_;
  Device* dev_;
  index_t p_, k_, r_;
};
using TruncatedPrecond = TruncatedPrecondT<double>;

/// spikes_T[i] = T_i (i = 0..p-2), spikes_W[i] = W_{i+1} (i = 0..p-2).
/// Throws IllConditionedInterfaceError(interface, cond_1) above cond_1 = 1e12.
template <class S>
std::shared_ptr<TruncatedPrecondT<S>> build_truncated_precond(
    const std::vector<LowRankSpikeT<S>>& spikes_T, const std::vector<LowRankSpikeT<S>>& spikes_W,
    index_t k, Device& dev = Device::default_device());
/// the Woodbury interface solves; first top / last bottom tips pass through.
template <class S>
ReducedVectorT<S> apply_truncated_precond(const TruncatedPrecondT<S>& P, const ReducedVectorT<S>& g);
/// x + the low-rank spike tips applied to the neighbour tips.
template <class S>
ReducedVectorT<S> matvec_lowrank(const TruncatedPrecondT<S>& P, const ReducedVectorT<S>& x);
template <class S>
ReducedVectorT<S> matvec_lowrank(const SpikeFactorizationT<S>& f, const ReducedVectorT<S>& x);
/// the exact reduced matvec with the spikes applied on the fly (padded
/// block solves); SPEC.md:340's matvec_exact computes the same operator from stored tips.
template <class S>
ReducedVectorT<S> matvec_otf(const SpikeFactorizationT<S>& f, const ReducedVectorT<S>& x);
template <class S>
ReducedVectorT<S> matvec_exact(const SpikeFactorizationT<S>& f, const ReducedVectorT<S>& x) {
  return matvec_otf(f, x);
}

/// SPEC.md:476-484 (r-halving retry on an ill-conditioned interface).
template <class S>
std::shared_ptr<SpikeFactorizationT<S>> factorize(const CsrMatrixT<S>& a, const SolverConfigT<S>& cfg,
                                                  Device& dev = Device::default_device());
/// The partition-sharded factorization: one process per GPU, every rank passes the full
/// matrix and the same config; applies and solves on it are collective over `comm`.
template <class S>
std::shared_ptr<SpikeFactorizationT<S>> factorize_dist(const CsrMatrixT<S>& a,
                                                       const SolverConfigT<S>& cfg,
                                                       Communicator& comm,
                                                       Device& dev = Device::default_device());
/// SPEC.md:485-493.
template <class S>
DenseBlockT<S> apply_precond_T(const SpikeFactorizationT<S>& f, const DenseBlockT<S>& rhs);
/// SPEC.md:494-502 (an LR_SPIKE_I factorization; inner BiCGStab on the reduced system).
template <class S>
DenseBlockT<S> apply_precond_I(const SpikeFactorizationT<S>& f, const DenseBlockT<S>& rhs);
/// SPEC.md:512-519.
template <class S>
DenseBlockT<S> apply_block_jacobi(const SpikeFactorizationT<S>& f, const DenseBlockT<S>& rhs);
/// factorize (or reuse f) and run the outer Krylov method.
/// Non-convergence is reported (report.converged == false), not thrown; a BiCGStab
/// breakdown throws BreakdownError carrying the partial solution.
template <class S>
std::pair<DenseBlockT<S>, SolveReport> solve(const CsrMatrixT<S>& a, const DenseBlockT<S>& rhs,
                                             const SolverConfigT<S>& cfg,
                                             std::shared_ptr<SpikeFactorizationT<S>> f = nullptr);

/// Operator contract of the Krylov drivers: out = Op(in) on device
/// blocks (n x n_rhs; the library's stream is synchronized before the call and the
/// callback must finish its work before returning).
template <class S>
using LinearOperatorT = std::function<void(DeviceView<const S> in, DeviceView<S> out)>;
using LinearOperator = LinearOperatorT<double>;
/// The SpMV of a device matrix / the preconditioner of a factorization as operators.
template <class S>
LinearOperatorT<S> as_operator(const DeviceMatrixT<S>& a);
template <class S>
LinearOperatorT<S> as_operator(const SpikeFactorizationT<S>& f);

/// SPEC.md:421-429 (right-preconditioned, half-iteration counts, true residual at
/// convergence, breakdown -> BreakdownError with the partial result); M may be null.
template <class S>
std::pair<DenseBlockT<S>, SolveReport> bicgstab(const LinearOperatorT<S>& A, const LinearOperatorT<S>* M,
                                                const DenseBlockT<S>& b, const IterConfigT<S>& it,
                                                Device& dev = Device::default_device());
/// SPEC.md:430-436 (A Hermitian positive definite).
template <class S>
std::pair<DenseBlockT<S>, SolveReport> cg(const LinearOperatorT<S>& A, const LinearOperatorT<S>* M,
                                          const DenseBlockT<S>& b, const IterConfigT<S>& it,
                                          Device& dev = Device::default_device());
/// Right-preconditioned restarted GMRES(it.restart) with CGS2 Arnoldi.
template <class S>
std::pair<DenseBlockT<S>, SolveReport> gmres(const LinearOperatorT<S>& A, const LinearOperatorT<S>* M,
                                             const DenseBlockT<S>& b, const IterConfigT<S>& it,
                                             Device& dev = Device::default_device());

}  // namespace lrspike

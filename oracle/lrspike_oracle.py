"""CPU ORACLE for the LR-SPIKE hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker / the CPU baseline.  The product path (liblrspike_cuda.so via
``paper_2504_11167_b200.api`` or ``include/lrspike``) never calls it.

What it restates.  The reference (/root/reference) implements only sparse_core
(proj/core/src/matrix.cpp); every solver operation exists only as a SPEC
contract.  This file restates those contracts in numpy/scipy,
citing the SPEC line each function follows, with LAPACK ``?gbtrf``/``?gbtrs``
(scipy's bundled OpenBLAS) standing in for the paper's PARDISO block solver
(SURVEY.md D3).  GMRES(m) is not in the reference (SPEC.md:452 lists it as a
non-goal) but BASELINE.json's configs require it; it is defined here once and
the CUDA path implements the identical algorithm.

Pinning.  The reference ships no tests, fixtures or golden vectors (SURVEY.md
section 0, fact 4) and cannot be built here (no Eigen; the solver is not
implemented), so ``oracle/_ref`` cannot exist.  The oracle is pinned instead
against every known-answer example in the SPEC ([TRIVIAL]/[DERIVED] examples
and the acceptance identities: Woodbury vs dense inverse, r=0 == Block
Jacobi, P=2 full-rank exactness, DS identity, ledger counts), see
tests/test_oracle.py and tests/golden/.  Against the paper's own (MKL/PARDISO)
implementation parity is unpinned; see DESIGN.md "Parity".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
from scipy.linalg import lapack

# --------------------------------------------------------------------------------------
# errors -- mirror of reference proj/core/include/lrspike/errors.hpp:11-94
# --------------------------------------------------------------------------------------


class Error(RuntimeError):
    """errors.hpp:11 ``lrspike::Error``."""


class DimensionError(Error):
    """errors.hpp:36."""


class LayoutError(Error):
    """errors.hpp:53: requested layout cannot satisfy n_i > k."""


class NotBlockTridiagonalError(Error):
    """errors.hpp:59-70, carries (row, col)."""

    def __init__(self, msg, row, col):
        super().__init__(msg)
        self.row, self.col = row, col


class SingularBlockError(Error):
    """errors.hpp:73-81, carries the column."""

    def __init__(self, msg, column):
        super().__init__(msg)
        self.column = column


class ParameterError(Error):
    """errors.hpp:83."""


class IllConditionedInterfaceError(Error):
    """errors.hpp:86-94, carries interface index and condition estimate."""

    def __init__(self, msg, interface_index, cond_estimate):
        super().__init__(msg)
        self.interface_index, self.cond_estimate = interface_index, cond_estimate


class BreakdownError(Error):
    """BiCGStab stagnation, carries the partial x and report."""

    def __init__(self, msg, x, report):
        super().__init__(msg)
        self.x, self.report = x, report


def _pmap(fn, *seqs):
    """list(map(fn, *seqs)) over LRS_ORACLE_THREADS host threads (default 1: sequential).
    Partitions and spikes are independent (results must not depend on the
    scheduling), and LAPACK releases the GIL, so the baseline runs partitions concurrently
    with OPENBLAS_NUM_THREADS=1; the results are identical."""
    import os

    t = int(os.environ.get("LRS_ORACLE_THREADS", "1") or 1)
    if t <= 1:
        return list(map(fn, *seqs))
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(t) as ex:
        return list(ex.map(fn, *seqs))


COND_LIMIT = 1e12  # interface condition limit; same constant on the GPU

# --------------------------------------------------------------------------------------
# sparse_core -- matrix.cpp:121-158
# --------------------------------------------------------------------------------------


def spmv(A: sp.csr_matrix, X: np.ndarray) -> np.ndarray:
    """matrix.cpp:121-136: Y = A X, ascending column order per row."""
    if A.shape[1] != X.shape[0]:
        raise DimensionError("spmv: A.n_cols must equal x.n_rows")
    return A @ X


def band_metrics(A: sp.csr_matrix):
    """matrix.cpp:138-158 -> (ku, kl, k, diag_weight, band_density)."""
    if A.shape[0] != A.shape[1]:
        raise DimensionError("band_metrics: matrix must be square")
    coo = A.tocoo()
    d = coo.col - coo.row
    ku = int(d.max(initial=0)) if d.size else 0
    kl = int((-d).max(initial=0)) if d.size else 0
    ku, kl = max(ku, 0), max(kl, 0)
    tot = float(np.abs(coo.data).sum())
    dia = float(np.abs(coo.data[d == 0]).sum())
    cells = (ku + kl + 1) * A.shape[0]
    return ku, kl, max(ku, kl), (dia / tot if tot > 0 else 0.0), (A.nnz / cells if cells else 0.0)


# --------------------------------------------------------------------------------------
# partition -- SPEC.md:152-204
# --------------------------------------------------------------------------------------


@dataclass
class PartitionLayout:
    p: int
    sizes: list
    offsets: list
    k: int


def make_layout(n: int, p: int, k: int) -> PartitionLayout:
    """first (n mod p) partitions get ceil(n/p) rows; n_i > k."""
    if p < 1 or k < 0:
        raise ParameterError("make_layout: p >= 1 and k >= 0 required")
    base, rem = divmod(n, p)
    sizes = [base + (1 if i < rem else 0) for i in range(p)]
    if min(sizes) <= k:
        raise LayoutError(f"layout infeasible: need n >= p*(k+1) = {p * (k + 1)}")
    offsets = [0]
    for s in sizes[:-1]:
        offsets.append(offsets[-1] + s)
    return PartitionLayout(p, sizes, offsets, k)


@dataclass
class PartitionBlocks:
    layout: PartitionLayout
    A: list  # csr n_i x n_i
    B: list  # csr k x k, B[i] couples partition i to i+1 (i = 0..p-2)
    C: list  # csr k x k, C[i] couples partition i to i-1 (i = 1..p-1); C[0] = None


def extract_blocks(A: sp.csr_matrix, lay: PartitionLayout) -> PartitionBlocks:
    """SPEC.md:180-188.  B_i = bottom-left k x k of the super-diagonal block,
    C_{i+1} = top-right of the sub-diagonal block (Eq. 6); any nonzero
    outside the block-tridiagonal pattern raises NotBlockTridiagonalError."""
    n = A.shape[0]
    if A.shape[0] != A.shape[1] or n != sum(lay.sizes):
        raise DimensionError("extract_blocks: A must be square and match the layout")
    k = lay.k
    part = np.repeat(np.arange(lay.p), lay.sizes)
    off = np.asarray(lay.offsets + [n])
    coo = A.tocoo()
    pr, pc = part[coo.row], part[coo.col]
    ok = pr == pc
    sup = pc == pr + 1
    ok |= sup & (coo.row >= off[pr + 1] - k) & (coo.col < off[np.minimum(pc, lay.p - 1)] + k)
    sub = pc == pr - 1
    ok |= sub & (coo.row < off[pr] + k) & (coo.col >= off[np.maximum(pr, 0)] - k)
    if not ok.all():
        bad = np.flatnonzero(~ok)
        # report the first offending entry in row-major order
        j = bad[np.lexsort((coo.col[bad], coo.row[bad]))[0]]
        r, c = int(coo.row[j]), int(coo.col[j])
        raise NotBlockTridiagonalError(
            f"nonzero ({r},{c}) outside the block-tridiagonal pattern; increase k or decrease p",
            r, c)
    As, Bs, Cs = [], [], [None]
    for i in range(lay.p):
        o, s = lay.offsets[i], lay.sizes[i]
        As.append(A[o:o + s, o:o + s].tocsr())
        if i + 1 < lay.p:
            o1 = lay.offsets[i + 1]
            Bs.append(A[o + s - k:o + s, o1:o1 + k].tocsr())
        if i > 0:
            om, sm = lay.offsets[i - 1], lay.sizes[i - 1]
            Cs.append(A[o:o + k, om + sm - k:om + sm].tocsr())
    return PartitionBlocks(lay, As, Bs, Cs)


# --------------------------------------------------------------------------------------
# block_solver -- SPEC.md:206-257 (banded LU with partial pivoting, LAPACK ?gbtrf, D3)
# --------------------------------------------------------------------------------------


@dataclass
class BlockFactor:
    n: int
    kl: int
    ku: int
    ab: np.ndarray  # LAPACK band storage (2kl+ku+1, n); the getrf n x n LU if dense
    ipiv: np.ndarray  # 0-based pivot rows
    dtype: np.dtype
    dense: bool = False  # ?getrf / ?getrs storage (see factorize_block)

    @property
    def swaps(self) -> int:
        return int(np.count_nonzero(self.ipiv != np.arange(self.n)))


def factorize_block(Ai: sp.csr_matrix, kl: int | None = None, ku: int | None = None) -> BlockFactor:
    """LU with partial pivoting (LAPACK dgbtrf semantics: first
    max |a| pivot, izamax |Re|+|Im| for complex); exact zero pivot ->
    SingularBlockError(column)."""
    n = Ai.shape[0]
    coo = Ai.tocoo()
    d = coo.col - coo.row
    if kl is None:
        kl = int(max(0, (-d).max(initial=0)))
    if ku is None:
        ku = int(max(0, d.max(initial=0)))
    dt = np.result_type(Ai.dtype, np.float64)
    if _dense_storage(n, kl, ku, np.dtype(dt).itemsize):
        a = np.asfortranarray(Ai.toarray().astype(dt))
        getrf, = lapack.get_lapack_funcs(("getrf",), (a,))
        lu, ipiv, info = getrf(a, overwrite_a=True)
        if info > 0:
            raise SingularBlockError(f"exact zero pivot in column {info - 1}", info - 1)
        if info < 0:
            raise ParameterError(f"getrf illegal argument {-info}")
        return BlockFactor(n, kl, ku, lu, ipiv, dt, True)
    ab = np.zeros((2 * kl + ku + 1, n), dtype=dt, order="F")
    ab[kl + ku + coo.row - coo.col, coo.col] = coo.data
    gbtrf, = lapack.get_lapack_funcs(("gbtrf",), (ab,))
    lu, ipiv, info = gbtrf(ab, kl, ku)
    if info > 0:
        raise SingularBlockError(f"exact zero pivot in column {info - 1}", info - 1)
    if info < 0:
        raise ParameterError(f"gbtrf illegal argument {-info}")
    return BlockFactor(n, kl, ku, lu, ipiv, dt)


def _dense_storage(n: int, kl: int, ku: int, itemsize: int) -> bool:
    """Store a block as a dense ?getrf LU when the band storage (2kl+ku+1) x n would be both
    larger than n x n and over 1 GiB (c3 at P = 64: 4.2 GB band vs 1.5 GB dense per block).
    Same factorization (LAPACK partial pivoting, first max |a| / izamax pivot, D3); only the
    storage and the blocking of the roundoff differ."""
    band = (2 * kl + ku + 1) * n * itemsize
    return band > n * n * itemsize and band > (1 << 30)


def _gbtrs(F: BlockFactor, R: np.ndarray, trans: int) -> np.ndarray:
    R = np.asarray(R)
    if R.shape[0] != F.n:
        raise DimensionError("solve_block: RHS rows must equal the block size")
    dt = np.result_type(F.dtype, R.dtype)
    vec = R.ndim == 1
    Rm = np.array(R.reshape(F.n, -1), dtype=dt, order="F")
    if Rm.shape[1] == 0:
        return Rm.reshape(R.shape)
    if F.dense:
        getrs, = lapack.get_lapack_funcs(("getrs",), (F.ab,))
        x, info = getrs(F.ab, F.ipiv, Rm, trans=trans)
    else:
        gbtrs, = lapack.get_lapack_funcs(("gbtrs",), (F.ab,))
        x, info = gbtrs(F.ab, F.kl, F.ku, Rm, F.ipiv, trans=trans)
    if info != 0:
        raise ParameterError(f"gbtrs failed {info}")
    return x.reshape(R.shape) if vec else x


def solve_block(F: BlockFactor, R: np.ndarray) -> np.ndarray:
    """A_i^-1 R, columns independent."""
    return _gbtrs(F, R, 0)


def solve_block_adjoint(F: BlockFactor, R: np.ndarray) -> np.ndarray:
    """A_i^-T R.  The SPEC is real-field; for the complex128
    config (c5) the field-generic adjoint is the conjugate
    transpose A_i^-H (gbtrs trans='C'), which is what the Halko range finder
    needs (T^H Q)."""
    return _gbtrs(F, R, 2 if np.iscomplexobj(F.ab) else 1)


# --------------------------------------------------------------------------------------
# spikes -- SPEC.md:259-321
# --------------------------------------------------------------------------------------

SIDE_T, SIDE_W = 0, 1


def _pad(coupling_times_x: np.ndarray, n: int, side: int) -> np.ndarray:
    k, c = coupling_times_x.shape
    R = np.zeros((n, c), dtype=coupling_times_x.dtype, order="F")
    if side == SIDE_T:
        R[n - k:] = coupling_times_x
    else:
        R[:k] = coupling_times_x
    return R


def compute_full_spike(F: BlockFactor, coupling, side: int) -> np.ndarray:
    """T_i = A_i^-1 [0; B_i] or W_i = A_i^-1 [C_i; 0]."""
    Cd = coupling.toarray() if sp.issparse(coupling) else np.asarray(coupling)
    if F.n < Cd.shape[0]:
        raise DimensionError("spike: block smaller than k")
    return solve_block(F, _pad(Cd, F.n, side))


@dataclass
class LowRankSpike:
    u: np.ndarray  # n_i x r, orthonormal columns
    sigma: np.ndarray  # r, non-increasing (collapsed entries set to 0)
    v: np.ndarray  # r x k, orthonormal rows
    side: int
    rank_collapsed: bool = False

    def tips(self, k):
        """(first k rows of u, last k rows of u)."""
        return self.u[:k], self.u[-k:]


def _orth(Y: np.ndarray) -> np.ndarray:
    """Householder QR, no column pivoting."""
    q, _ = np.linalg.qr(Y, mode="reduced")
    return q


def randomized_spike_svd(F: BlockFactor, coupling, side: int, n_svd: int, oversample: int,
                         passes: int, seed: int, partition: int) -> LowRankSpike:
    """SPEC.md:286-294 (Halko-Martinsson-Tropp proto-algorithm, matrix-free).

    Omega ~ N(0,1)^{k x l} from stream (seed, partition, side);
    Y = T Omega by one padded solve; Q = orth(Y); each extra pair of passes
    Q = orth(T orth(T^T Q)); Z^T = T^T Q = coupling^T (A_i^-T Q)|tip; SVD(Z);
    u = Q U[:, :r], sigma = s[:r], v = V[:r].  Rank collapse sigma_j <
    1e-14 sigma_1 zeroes those sigma_j and sets the warning flag.
    """
    Cs = coupling.tocsr() if sp.issparse(coupling) else sp.csr_matrix(coupling)
    k = Cs.shape[0]
    l = n_svd + oversample
    if n_svd < 1 or n_svd > k:
        raise ParameterError("randomized_spike_svd: 1 <= n_svd <= k required")
    if oversample < 0 or l > k:
        raise ParameterError("randomized_spike_svd: n_svd + oversample <= k required")
    if passes < 2:
        raise ParameterError("randomized_spike_svd: passes >= 2 required")
    n = F.n
    Om = omega_block(seed, partition, side, k, l)

    def T_apply(X):
        return solve_block(F, _pad(np.asarray(Cs @ X), n, side))

    CsH = Cs.conj().T if np.iscomplexobj(Cs.data) else Cs.T

    def Tt_apply(Q):  # T^H Q (T^T Q for real)
        S = solve_block_adjoint(F, Q)
        tip = S[n - k:] if side == SIDE_T else S[:k]
        return np.asarray(CsH @ tip)

    Q = _orth(T_apply(Om))
    for _ in range((passes - 2) // 2):
        W = _orth(Tt_apply(Q))
        Q = _orth(T_apply(W))
    Zt = Tt_apply(Q)  # k x l, = (Q^H T)^H
    Uh, s, Vh = np.linalg.svd(Zt.conj().T, full_matrices=False)  # Z = Uh diag(s) Vh
    u = Q @ Uh[:, :n_svd]
    sigma = s[:n_svd].copy()
    v = Vh[:n_svd].copy()
    collapsed = False
    if sigma.size and (sigma[0] == 0 or np.any(sigma < 1e-14 * sigma[0])):
        collapsed = True
        sigma[sigma < 1e-14 * sigma[0]] = 0.0
        if s[0] == 0:
            sigma[:] = 0.0
    return LowRankSpike(u, sigma, v, side, collapsed)


def coupling_spike_svd(F: BlockFactor, coupling, side: int, n_svd: int, oversample: int,
                       passes: int, seed: int, partition: int) -> LowRankSpike:
    """spike_mode = "coupling" (BASELINE.json north_star setup (1): "truncated rank-k SVD of
    B_j and C_j ... form the low-rank spikes by multi-RHS solves against the k singular
    vectors"; the construction the paper compares against at PAPER.md:939-943, :1272-1276
    and SPEC acceptance 6).

    Rank-r randomized SVD of the k x k coupling block (Halko range finder with exactly r
    columns -- the first r columns of the spike mode's Omega stream -- and (passes - 2) / 2
    power iterations):  Q_B = orth(B Omega_r),  Z^H = B^H Q_B,  Z = U^ S V^H, so
    B_r = U_B S_B V_B^H with U_B = Q_B U^.  B_r = Q_B Q_B^H B is fixed by span(B Omega_r)
    even when B's spectrum is flat (B ~ -I for the natural-ordered stencils), so no tie
    among equal singular values decides the result.  The spike is
    T~ = A_i^-1 pad(U_B S_B) V_B^H (r padded solves), returned in the LowRankSpike form
    (orthonormal u, non-increasing sigma, orthonormal v) through Y = Q2 R2,
    R2 = U2 S2 V2^H:  u = Q2 U2, sigma = S2, v = V2^H V_B^H."""
    Cs = coupling.tocsr() if sp.issparse(coupling) else sp.csr_matrix(coupling)
    k = Cs.shape[0]
    l = n_svd + oversample
    if n_svd < 1 or n_svd > k:
        raise ParameterError("coupling_spike_svd: 1 <= n_svd <= k required")
    if oversample < 0 or l > k:
        raise ParameterError("coupling_spike_svd: n_svd + oversample <= k required")
    if passes < 2:
        raise ParameterError("coupling_spike_svd: passes >= 2 required")
    Om = omega_block(seed, partition, side, k, l)[:, :n_svd]
    CsH = Cs.conj().T if np.iscomplexobj(Cs.data) else Cs.T
    QB = _orth(np.asarray(Cs @ Om))
    for _ in range((passes - 2) // 2):
        QB = _orth(np.asarray(Cs @ _orth(np.asarray(CsH @ QB))))
    Zt = np.asarray(CsH @ QB)  # k x r = (Q_B^H B)^H
    Uh, sB, VBh = np.linalg.svd(Zt.conj().T, full_matrices=False)  # Z = Uh diag(sB) VBh
    UB = QB @ Uh
    Y = solve_block(F, _pad(UB * sB, F.n, side))
    Q2, R2 = np.linalg.qr(Y, mode="reduced")
    U2, s2, V2h = np.linalg.svd(R2)
    u = Q2 @ U2
    sigma = s2.copy()
    v = V2h @ VBh
    collapsed = False
    if sigma.size and (sigma[0] == 0 or np.any(sigma < 1e-14 * sigma[0])):
        collapsed = True
        sigma[sigma < 1e-14 * sigma[0]] = 0.0
        if s2[0] == 0:
            sigma[:] = 0.0
    return LowRankSpike(u, sigma, v, side, collapsed)


def omega_block(seed, partition, side, rows, cols):
    from paper_2504_11167_b200 import configs  # the shared input generator (not the product)

    return configs.omega(seed, partition, side, rows, cols)


# --------------------------------------------------------------------------------------
# reduced_system -- SPEC.md:323-404, Appendix A of SURVEY.md
# --------------------------------------------------------------------------------------


@dataclass
class CommLedger:
    """per stage messages and scalars."""

    stages: dict = field(default_factory=dict)

    def record(self, stage, messages, scalars):
        m, s = self.stages.get(stage, (0, 0))
        self.stages[stage] = (m + messages, s + scalars)


@dataclass
class Interface:
    degenerate: bool
    uTb: np.ndarray  # k x r  (last k rows of u_{T_i})
    sT: np.ndarray
    vT: np.ndarray  # r x k
    uWt: np.ndarray  # k x r  (first k rows of u_{W_{i+1}})
    sW: np.ndarray
    vW: np.ndarray
    G: np.ndarray | None = None  # (vW uTb)^-1 explicit
    E: np.ndarray | None = None  # vT uWt
    H_lu: tuple | None = None
    cond: float = 1.0


@dataclass
class TruncatedPrecond:
    k: int
    r: int
    interfaces: list


def _cond1(M: np.ndarray) -> float:
    try:
        inv = np.linalg.inv(M)
    except np.linalg.LinAlgError:
        return math.inf
    c = float(np.abs(M).sum(0).max() * np.abs(inv).sum(0).max())
    return c if np.isfinite(c) else math.inf


def build_truncated_precond(spT: list, spW: list, k: int) -> TruncatedPrecond:
    """SPEC.md:367-375 (paper Eq. red_sys_prec_inv): per interface i=0..p-2,
    G_i = (vW_{i+1} uT_{i,b})^-1 explicit, H_i = G_i - S_T vT uW_{i+1,t} S_W, LU(H_i).
    Interfaces where either spike has all-zero sigma are the identity (M_i = I).
    cond_1 > COND_LIMIT -> IllConditionedInterfaceError(i, cond)."""
    ifs = []
    r = spT[0].sigma.size if spT else 0
    for i in range(len(spT)):
        sT, sW = spT[i], spW[i + 1]
        it = Interface(False, sT.u[-k:], sT.sigma, sT.v, sW.u[:k], sW.sigma, sW.v)
        if not np.any(sT.sigma) or not np.any(sW.sigma):
            it.degenerate = True
            ifs.append(it)
            continue
        K = sW.v @ sT.u[-k:]
        cK = _cond1(K)
        if cK > COND_LIMIT:
            raise IllConditionedInterfaceError(f"interface {i}: cond(K)={cK:.3e}", i, cK)
        G = np.linalg.inv(K)
        E = sT.v @ sW.u[:k]
        H = G - (sT.sigma[:, None] * E) * sW.sigma[None, :]
        cH = _cond1(H)
        if cH > COND_LIMIT:
            raise IllConditionedInterfaceError(f"interface {i}: cond(H)={cH:.3e}", i, cH)
        it.G, it.E, it.H_lu, it.cond = G, E, sla.lu_factor(H), cH
        ifs.append(it)
    return TruncatedPrecond(k, r, ifs)


def apply_truncated_precond(P: TruncatedPrecond, top: list, bot: list, ledger=None):
    """SPEC.md:376-385 via Appendix A.1 (W1-W4).  ``top[i]``/``bot[i]`` are the
    k x n_rhs tips g_{i,t}, g_{i,b}; returns the reduced solution tips."""
    p = len(top)
    xt = [t.copy() for t in top]
    xb = [b.copy() for b in bot]
    for i, it in enumerate(P.interfaces):
        gb, gt = bot[i], top[i + 1]
        if it.degenerate:
            # M_i = I: x_{i+1,t} = g_{i+1,t} - W g_{i,b}; x_{i,b} = g_{i,b} - T x_{i+1,t}
            xt[i + 1] = gt - it.uWt @ (it.sW[:, None] * (it.vW @ gb))
            xb[i] = gb - it.uTb @ (it.sT[:, None] * (it.vT @ xt[i + 1]))
        else:
            mW = it.vW @ gb  # W1 message  i -> i+1
            mT = it.vT @ gt  # W1 message  i+1 -> i
            vTz = mT - it.E @ (it.sW[:, None] * mW)
            h = sla.lu_solve(it.H_lu, it.sT[:, None] * vTz)
            z = gt - it.uWt @ (it.sW[:, None] * mW)  # W2
            xt[i + 1] = z + it.uWt @ (it.sW[:, None] * h)
            vTMz = vTz + it.E @ (it.sW[:, None] * h)  # W3
            xb[i] = gb - it.uTb @ (it.sT[:, None] * vTMz)
        if ledger is not None:
            ledger.record("precond-apply", 2, 2 * P.r * gb.shape[1])
    del p
    return xt, xb


def matvec_exact(tipsT: list, tipsW: list, xt: list, xb: list):
    """SPEC.md:340-348 (Eqs. 19-21): y_i = x_i + W_tips x_{i-1,b} + T_tips x_{i+1,t}.
    tipsT[i] = (T_{i,t}, T_{i,b}) for i=0..p-2; tipsW[i] = (W_{i,t}, W_{i,b}) for i=1..p-1."""
    p = len(xt)
    yt = [a.copy() for a in xt]
    yb = [a.copy() for a in xb]
    for i in range(p):
        if i > 0:
            Wt, Wb = tipsW[i]
            yt[i] += Wt @ xb[i - 1]
            yb[i] += Wb @ xb[i - 1]
        if i < p - 1:
            Tt, Tb = tipsT[i]
            yt[i] += Tt @ xt[i + 1]
            yb[i] += Tb @ xt[i + 1]
    return yt, yb


# --------------------------------------------------------------------------------------
# spike_solvers -- SPEC.md:457-549
# --------------------------------------------------------------------------------------


@dataclass
class SolverConfig:
    """SPEC.md:470-473 (outer IterConfig is passed to solve separately).

    variant: "T" (LR-SPIKE-T), "I" (LR-SPIKE-I), "OTF" (LR-SPIKE-OTF), "BJ" (Block
    Jacobi).  inner: the LR-SPIKE-I reduced solve (SPEC.md:472 names 1e-16 after the
    paper's Table 3; a BiCGStab true residual cannot certify 1e-16 in FP64, so the
    default here is 1e-12); otf_tol / otf_escalations: LR-SPIKE-OTF's reduced-system
    tolerance and its escalation schedule (/100 per escalation, at most 4)."""

    variant: str = "T"
    p: int = 4
    k: int | None = None  # None -> band_metrics(A).k
    n_svd: int = 8
    oversample: int | None = None  # None -> ceil(n_svd/2)
    passes: int = 2
    seed: int = 0
    inner_tol: float = 1e-12
    inner_max_iters: int = 200
    otf_tol: float = 1e-8
    otf_max_iters: int = 500
    otf_escalations: int = 4
    factor_fp32: bool = False  # FP32 off-diagonal factor tiles in the applies
    # "spike": randomized SVD of the spike T_i = A_i^-1 [0; B_i] (default);
    # "coupling": truncated SVD of B_i / C_i, spikes by multi-RHS solves against the
    # singular vectors (BASELINE.json north_star setup (1))
    spike_mode: str = "spike"


@dataclass
class SpikeFactorization:
    blocks: PartitionBlocks
    factors: list
    spT: list
    spW: list
    trunc: TruncatedPrecond | None
    cfg: SolverConfig
    n_svd: int
    ledger: CommLedger = field(default_factory=CommLedger)
    rank_collapsed: bool = False
    inner_iterations: float = 0.0  # LR-SPIKE-I: inner half-iterations summed over applies
    inner_solves: int = 0
    factors32: list | None = None  # the applies' factors with FP32 off-diagonal tiles

    def apply_factors(self):
        return self.factors32 if self.factors32 is not None else self.factors


def factorize(A: sp.csr_matrix, cfg: SolverConfig) -> SpikeFactorization:
    """layout -> blocks -> per-partition LU -> randomized spike
    SVDs -> truncated preconditioner; on IllConditionedInterfaceError halve
    n_svd once, then fail."""
    A = sp.csr_matrix(A)
    k = cfg.k if cfg.k is not None else band_metrics(A)[2]
    lay = make_layout(A.shape[0], cfg.p, k)
    blocks = extract_blocks(A, lay)
    factors = _pmap(factorize_block, blocks.A)
    if cfg.variant not in ("T", "I", "OTF", "BJ"):
        raise ParameterError(f"unknown variant {cfg.variant!r}")
    n_svd = cfg.n_svd if cfg.variant in ("T", "I", "OTF") else 0
    for attempt in range(2):
        spT, spW, trunc, coll = _build_spikes(blocks, factors, cfg, n_svd, k)
        try:
            if n_svd > 0:
                trunc = build_truncated_precond(spT, spW, k)
            break
        except IllConditionedInterfaceError:
            if attempt == 1 or n_svd // 2 < 1:
                raise
            n_svd //= 2
    F = SpikeFactorization(blocks, factors, spT, spW, trunc, cfg, n_svd, rank_collapsed=coll)
    if cfg.factor_fp32:
        F.factors32 = [round_offdiag_tiles(fo) for fo in factors]
    return F


TILE = 128  # the GPU's factor tile (csrc/lrs_internal.h NB)


def round_offdiag_tiles(F: BlockFactor) -> BlockFactor:
    """The mixed-precision apply's factors (the paper applies single-precision
    preconditioners, section 4.3): L / U entries (i, j) outside the 128 x 128 diagonal tiles
    rounded to FP32 (the GPU keeps those tiles in FP32 and the diagonal-tile inverses in
    FP64).  Band storage: ab[kl + ku + i - j, j] holds entry (i, j)."""
    if F.dense:
        raise ParameterError("factor_fp32 emulation needs band storage")
    ab = F.ab.copy()
    kv = F.kl + F.ku
    rows, cols = np.indices(ab.shape)
    i = rows - kv + cols
    mask = (rows >= F.kl) & (i >= 0) & (i < F.n) & ((i // TILE) != (cols // TILE))
    ab[mask] = ab[mask].astype(np.float32).astype(ab.dtype)
    return BlockFactor(F.n, F.kl, F.ku, ab, F.ipiv, F.dtype)


def _build_spikes(blocks, factors, cfg, n_svd, k):
    p = blocks.layout.p
    if n_svd == 0 or p == 1:
        return [], [None] * p, None, False
    os_ = cfg.oversample if cfg.oversample is not None else (n_svd + 1) // 2
    if cfg.spike_mode not in ("spike", "coupling"):
        raise ParameterError(f"unknown spike_mode {cfg.spike_mode!r}")
    svd = randomized_spike_svd if cfg.spike_mode == "spike" else coupling_spike_svd
    spT = _pmap(lambda i: svd(factors[i], blocks.B[i], SIDE_T, n_svd, os_, cfg.passes,
                              cfg.seed, i), range(p - 1))
    spW = [None] + _pmap(lambda i: svd(factors[i], blocks.C[i], SIDE_W, n_svd, os_, cfg.passes,
                                       cfg.seed, i), range(1, p))
    coll = any(s.rank_collapsed for s in spT) or any(s.rank_collapsed for s in spW[1:])
    return spT, spW, None, coll


def _split(F: SpikeFactorization, f: np.ndarray):
    lay = F.blocks.layout
    return [f[o:o + s] for o, s in zip(lay.offsets, lay.sizes)]


def apply_block_jacobi(F: SpikeFactorization, f: np.ndarray) -> np.ndarray:
    """D^-1 f, no communication."""
    f2 = f.reshape(f.shape[0], -1)
    y = np.concatenate(_pmap(solve_block, F.apply_factors(), _split(F, f2)))
    return y.reshape(f.shape)


def apply_precond_T(F: SpikeFactorization, f: np.ndarray) -> np.ndarray:
    """y = D^-1 f; tips -> apply_truncated_precond -> low-rank
    recovery x_i = y_i - uW SW (vW x_{i-1,b}) - uT ST (vT x_{i+1,t})."""
    if F.n_svd == 0 or F.trunc is None:
        return apply_block_jacobi(F, f)
    f2 = f.reshape(f.shape[0], -1)
    k = F.blocks.layout.k
    ys = _pmap(solve_block, F.apply_factors(), _split(F, f2))
    top = [y[:k] for y in ys]
    bot = [y[-k:] for y in ys]
    xt, xb = apply_truncated_precond(F.trunc, top, bot, F.ledger)
    return _lowrank_recovery(F, ys, xt, xb, f2.shape[1]).reshape(f.shape)


def _pack(xt, xb):
    """ReducedVector as one 2kp x n_rhs block: partition i's top tip
    in rows [2ki, 2ki+k), its bottom tip in [2ki+k, 2k(i+1))."""
    return np.concatenate([np.concatenate([t, b]) for t, b in zip(xt, xb)])


def _unpack(v, p, k):
    v = v.reshape(v.shape[0], -1)
    return ([v[2 * k * i:2 * k * i + k] for i in range(p)],
            [v[2 * k * i + k:2 * k * (i + 1)] for i in range(p)])


def matvec_lowrank(F: SpikeFactorization, xt: list, xb: list, ledger=None):
    """y_i = x_i + W~_i x_{i-1,b} + T~_i x_{i+1,t} with the low-rank
    spikes: the owner of x_{i-1,b} sends the compressed message S_W v_W x_{i-1,b}
    (r x n_rhs), the owner of x_{i+1,t} sends S_T v_T x_{i+1,t}; the receiver applies
    its u tips (top k and bottom k rows).  W term first, then T term."""
    p = len(xt)
    k = F.blocks.layout.k
    yt = [a.copy() for a in xt]
    yb = [a.copy() for a in xb]
    nr = xt[0].shape[1]
    for i in range(p):
        if i > 0:
            s = F.spW[i]
            m = s.sigma[:, None] * (s.v @ xb[i - 1])
            yt[i] = yt[i] + s.u[:k] @ m
            yb[i] = yb[i] + s.u[-k:] @ m
            if ledger is not None:
                ledger.record("reduced-matvec", 1, F.n_svd * nr)
        if i < p - 1:
            s = F.spT[i]
            m = s.sigma[:, None] * (s.v @ xt[i + 1])
            yt[i] = yt[i] + s.u[:k] @ m
            yb[i] = yb[i] + s.u[-k:] @ m
            if ledger is not None:
                ledger.record("reduced-matvec", 1, F.n_svd * nr)
    return yt, yb


def _coupled_solve(F: SpikeFactorization, xt: list, xb: list, nr: int):
    """z_i = A_i^-1 (pad_top(C_i x_{i-1,b}) + pad_bottom(B_i x_{i+1,t})) = W_i x_{i-1,b}
    + T_i x_{i+1,t} with the exact spikes (padded solve_block)."""
    lay = F.blocks.layout
    k, p = lay.k, lay.p
    zs = []
    for i in range(p):
        n_i = lay.sizes[i]
        dt = np.result_type(xt[0].dtype, F.factors[i].dtype)
        rhs = np.zeros((n_i, nr), dtype=dt)
        if i > 0:
            rhs[:k] += np.asarray(F.blocks.C[i] @ xb[i - 1])
        if i < p - 1:
            rhs[n_i - k:] += np.asarray(F.blocks.B[i] @ xt[i + 1])
        zs.append(solve_block(F.apply_factors()[i], rhs))
    return zs


def matvec_otf(F: SpikeFactorization, xt: list, xb: list, ledger=None):
    """the TRUE reduced matvec, tips of the exact spikes evaluated on
    the fly (right to left: couplings, padded block solve, first/last k rows); the
    messages are the uncompressed k x n_rhs neighbour tips."""
    p = len(xt)
    k = F.blocks.layout.k
    nr = xt[0].shape[1]
    zs = _coupled_solve(F, xt, xb, nr)
    if ledger is not None and p > 1:
        ledger.record("reduced-matvec", 2 * (p - 1), 2 * (p - 1) * k * nr)
    return ([xt[i] + zs[i][:k] for i in range(p)], [xb[i] + zs[i][-k:] for i in range(p)])


def _lowrank_recovery(F, ys, xt, xb, nr):
    p = len(ys)
    out = []
    for i, y in enumerate(ys):
        x = y.copy()
        if i > 0:
            s = F.spW[i]
            x -= s.u @ (s.sigma[:, None] * (s.v @ xb[i - 1]))
            F.ledger.record("recovery", 1, F.n_svd * nr)
        if i < p - 1:
            s = F.spT[i]
            x -= s.u @ (s.sigma[:, None] * (s.v @ xt[i + 1]))
            F.ledger.record("recovery", 1, F.n_svd * nr)
        out.append(x)
    return np.concatenate(out)


class PreconditionerFailureError(Error):
    """LR-SPIKE-I inner reduced solve did not converge; carries the
    inner SolveReport."""

    def __init__(self, msg, report):
        super().__init__(msg)
        self.report = report


def apply_precond_I(F: SpikeFactorization, f: np.ndarray) -> np.ndarray:
    """D-stage; inner BiCGStab on the low-rank reduced system S~_r
    (operator matvec_lowrank, preconditioner apply_truncated_precond, tolerance
    cfg.inner_tol); recovery with the low-rank spikes as in apply_precond_T.  Inner
    iterations are accumulated on F (reported with the outer solve)."""
    if F.n_svd == 0 or F.trunc is None:
        return apply_block_jacobi(F, f)
    f2 = f.reshape(f.shape[0], -1)
    lay = F.blocks.layout
    k, p = lay.k, lay.p
    ys = _pmap(solve_block, F.apply_factors(), _split(F, f2))
    g = _pack([y[:k] for y in ys], [y[-k:] for y in ys])
    # the inner solve runs on the column-normalised reduced right-hand side (and scales
    # back): the reduced system is linear, and the absolute breakdown threshold then
    # does not fire on the tiny residuals an outer solve applies M to near convergence
    gn = _cnorm(g)
    gs = np.where(gn > 0, gn, 1.0)
    A_r = lambda v: _pack(*matvec_lowrank(F, *_unpack(v, p, k), F.ledger))  # noqa: E731
    M_r = lambda v: _pack(*apply_truncated_precond(F.trunc, *_unpack(v, p, k), F.ledger))  # noqa: E731
    icfg = IterConfig(tol=F.cfg.inner_tol, max_iters=F.cfg.inner_max_iters)
    try:
        xr, rep = bicgstab(A_r, M_r, g / gs, icfg)
        xr = xr * gs
    except BreakdownError as e:
        raise PreconditionerFailureError("LR-SPIKE-I inner solve broke down", e.report)
    if not rep.converged:
        raise PreconditionerFailureError("LR-SPIKE-I inner solve did not converge", rep)
    F.inner_iterations += rep.iterations
    F.inner_solves += 1
    xt, xb = _unpack(xr, p, k)
    return _lowrank_recovery(F, ys, xt, xb, f2.shape[1]).reshape(f.shape)


def solve_otf(A: sp.csr_matrix, F: SpikeFactorization, f: np.ndarray, it: "IterConfig"):
    """D-stage once; BiCGStab on the TRUE reduced system (matvec_otf)
    preconditioned by apply_truncated_precond to cfg.otf_tol; exact recovery
    x_i = y_i - A_i^-1 (pad_top(C_i x_{i-1,b}) + pad_bottom(B_i x_{i+1,t})); if the full
    relative residual misses it.tol, the reduced tolerance is divided by 100 and the
    reduced solve restarts warm from the previous x_r, at most cfg.otf_escalations
    times; exhausted -> the last x with converged = False.  iterations = reduced
    BiCGStab half-iterations summed over the escalations."""
    f2 = np.asarray(f).reshape(f.shape[0], -1)
    lay = F.blocks.layout
    k, p = lay.k, lay.p
    nr = f2.shape[1]
    ys = _pmap(solve_block, F.apply_factors(), _split(F, f2))
    g = _pack([y[:k] for y in ys], [y[-k:] for y in ys])
    rep = SolveReport()
    rep.precond_applications = 1  # the D-stage
    bn = _cnorm(f2)
    bn_safe = np.where(bn > 0, bn, 1.0)
    if F.n_svd == 0 or F.trunc is None or p == 1:
        M_r = lambda v: v  # noqa: E731
    else:
        M_r = lambda v: _pack(*apply_truncated_precond(F.trunc, *_unpack(v, p, k), F.ledger))  # noqa: E731
    A_r = lambda v: _pack(*matvec_otf(F, *_unpack(v, p, k), F.ledger))  # noqa: E731
    if p == 1 or all(B.nnz == 0 for B in F.blocks.B) and all(C.nnz == 0 for C in F.blocks.C[1:]):
        # no coupling: S_r = I, x = D^-1 f with zero reduced iterations
        x = np.concatenate(ys)
        rep.residual_final = float(np.max(_cnorm(f2 - A @ x) / bn_safe))
        rep.converged = bool(rep.residual_final <= it.tol)
        return x.reshape(np.asarray(f).shape), rep
    tol = F.cfg.otf_tol
    xr0 = None
    x = None
    total = 0.0
    for esc in range(F.cfg.otf_escalations + 1):
        rcfg = IterConfig(tol=tol, max_iters=F.cfg.otf_max_iters,
                          breakdown_eps=it.breakdown_eps, initial_guess=xr0)
        xr, rr = bicgstab(A_r, M_r, g, rcfg)
        total += rr.iterations
        rep.matvecs += rr.matvecs
        rep.residual_history.extend(rr.residual_history)
        xt, xb = _unpack(xr, p, k)
        zs = _coupled_solve(F, xt, xb, nr)
        if p > 1:
            F.ledger.record("recovery", 2 * (p - 1), 2 * (p - 1) * k * nr)
        x = np.concatenate([ys[i] - zs[i] for i in range(p)])
        res = _cnorm(f2 - A @ x) / bn_safe
        rep.matvecs += 1
        if np.all(res <= it.tol):
            rep.converged = True
            break
        tol /= 100.0
        xr0 = xr
    rep.iterations = total
    rep.residual_final = float(np.max(_cnorm(f2 - A @ x) / bn_safe))
    return x.reshape(np.asarray(f).shape), rep


# --------------------------------------------------------------------------------------
# krylov -- SPEC.md:406-455 (+ GMRES(m), D1)
# --------------------------------------------------------------------------------------


@dataclass
class IterConfig:
    """SPEC.md:411-414."""

    tol: float = 1e-8
    max_iters: int = 1000
    breakdown_eps: float = 1e-30
    initial_guess: np.ndarray | None = None
    restart: int = 30  # GMRES(m)


@dataclass
class SolveReport:
    """SPEC.md:415-419 (+ per-column iterations)."""

    converged: bool = False
    iterations: float = 0.0
    col_iterations: list = field(default_factory=list)
    residual_history: list = field(default_factory=list)
    precond_applications: int = 0
    matvecs: int = 0
    residual_final: float = math.nan
    breakdown: bool = False
    inner_iterations: float = 0.0  # LR-SPIKE-I inner half-iterations (summed)


def _cnorm(X):
    return np.sqrt(np.sum(np.abs(X) ** 2, axis=0))


def _cdot(X, Y):
    return np.sum(np.conj(X) * Y, axis=0)


def bicgstab(apply_A, apply_M, b: np.ndarray, cfg: IterConfig):
    """right-preconditioned BiCGStab, columns independent but
    batched, half-iteration granularity, true residual recomputed
    at claimed convergence; |rho| or |omega| < eps ->
    BreakdownError with the partial result.

    Convergence test at a half step (s) and a full step (r): estimate <= tol ->
    recompute ||b - A x|| / ||b||; accept only if that is <= tol, otherwise
    continue with the recursive residual."""
    b = np.asarray(b).reshape(b.shape[0], -1)
    n, nc = b.shape
    dt = np.result_type(b.dtype, np.float64)
    rep = SolveReport()
    bn = _cnorm(b)
    bn_safe = np.where(bn > 0, bn, 1.0)
    if cfg.initial_guess is not None:
        x = np.array(cfg.initial_guess, dtype=dt).reshape(n, nc)
        r = b - apply_A(x)
        rep.matvecs += 1
    else:
        x = np.zeros((n, nc), dtype=dt)
        r = b.astype(dt, copy=True)
    conv = _cnorm(r) / bn_safe <= cfg.tol
    conv |= bn == 0
    iters = np.zeros(nc)
    rep.residual_history.append(float(np.max(_cnorm(r) / bn_safe)))
    rhat = r.copy()
    rho_prev = np.ones(nc, dtype=dt)
    alpha = np.ones(nc, dtype=dt)
    omega = np.ones(nc, dtype=dt)
    p = np.zeros((n, nc), dtype=dt)
    v = np.zeros((n, nc), dtype=dt)
    brk = np.zeros(nc, dtype=bool)
    for it in range(1, cfg.max_iters + 1):
        act = ~conv & ~brk
        if not act.any():
            break
        rho = _cdot(rhat, r)
        brk |= act & (np.abs(rho) < cfg.breakdown_eps)
        act &= ~brk
        if not act.any():
            break
        if it == 1:
            p[:, act] = r[:, act]
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            p[:, act] = r[:, act] + beta[act] * (p[:, act] - omega[act] * v[:, act])
        phat = apply_M(p)
        v = np.where(act, apply_A(phat), v)
        rep.precond_applications += 1
        rep.matvecs += 1
        rv = _cdot(rhat, v)
        alpha = np.where(act, rho / np.where(rv != 0, rv, 1.0), alpha)
        s = np.where(act, r - alpha * v, r)
        sres = _cnorm(s) / bn_safe
        half = act & (sres <= cfg.tol)
        if half.any():
            xh = x + alpha * phat
            tr = _cnorm(b - apply_A(xh)) / bn_safe
            rep.matvecs += 1
            ok = half & (tr <= cfg.tol)
            x[:, ok] = xh[:, ok]
            conv |= ok
            iters[ok] = it - 0.5
            act &= ~ok
        rep.residual_history.append(float(np.max(np.where(act | half, sres, 0.0))))
        if not act.any():
            break
        shat = apply_M(s)
        t = np.where(act, apply_A(shat), 0)
        rep.precond_applications += 1
        rep.matvecs += 1
        tt = _cdot(t, t)
        om = _cdot(t, s) / np.where(tt != 0, tt, 1.0)
        omega = np.where(act, om, omega)
        brk |= act & (np.abs(omega) < cfg.breakdown_eps)
        act &= ~brk
        x[:, act] = x[:, act] + alpha[act] * phat[:, act] + omega[act] * shat[:, act]
        r[:, act] = s[:, act] - omega[act] * t[:, act]
        rres = _cnorm(r) / bn_safe
        full = act & (rres <= cfg.tol)
        if full.any():
            tr = _cnorm(b - apply_A(x)) / bn_safe
            rep.matvecs += 1
            ok = full & (tr <= cfg.tol)
            conv |= ok
            iters[ok] = it
        rep.residual_history.append(float(np.max(np.where(act, rres, 0.0))))
        rho_prev = np.where(act, rho, rho_prev)
        iters[act & ~conv] = it
    rep.col_iterations = iters.tolist()
    rep.iterations = float(iters.max()) if nc else 0.0
    rep.converged = bool(conv.all())
    rep.residual_final = float(np.max(_cnorm(b - apply_A(x)) / bn_safe))
    rep.breakdown = bool(brk.any())
    if brk.any():
        raise BreakdownError("BiCGStab stagnation detected (SF)", x, rep)
    return x, rep


def cg(apply_A, apply_M, b: np.ndarray, cfg: IterConfig):
    """preconditioned CG (A Hermitian positive definite, trusted).
    Columns independent but batched, like bicgstab.  The iteration count is in
    BiCGStab half-iteration units -- 0.5 per CG step, i.e. one unit per two
    preconditioner applications -- so A = I converges at 0.5.
    Convergence of the recursive residual triggers a true-residual check
    (SPEC.md:424's contract); |p^H A p| or |r^H z| < breakdown_eps -> BreakdownError."""
    b = np.asarray(b).reshape(b.shape[0], -1)
    n, nc = b.shape
    dt = np.result_type(b.dtype, np.float64)
    rep = SolveReport()
    bn = _cnorm(b)
    bn_safe = np.where(bn > 0, bn, 1.0)
    if cfg.initial_guess is not None:
        x = np.array(cfg.initial_guess, dtype=dt).reshape(n, nc)
        r = b - apply_A(x)
        rep.matvecs += 1
    else:
        x = np.zeros((n, nc), dtype=dt)
        r = b.astype(dt, copy=True)
    conv = (_cnorm(r) / bn_safe <= cfg.tol) | (bn == 0)
    rep.residual_history.append(float(np.max(_cnorm(r) / bn_safe)))
    iters = np.zeros(nc)
    brk = np.zeros(nc, dtype=bool)
    z = apply_M(r)
    rep.precond_applications += 1
    p = z.copy()
    rz = _cdot(r, z)
    for it in range(1, cfg.max_iters + 1):
        act = ~conv & ~brk
        if not act.any():
            break
        brk |= act & (np.abs(rz) < cfg.breakdown_eps)
        act &= ~brk
        if not act.any():
            break
        q = apply_A(p)
        rep.matvecs += 1
        pq = _cdot(p, q)
        brk |= act & (np.abs(pq) < cfg.breakdown_eps)
        act &= ~brk
        if not act.any():
            break
        alpha = np.where(act, rz / np.where(pq != 0, pq, 1.0), 0.0)
        x = np.where(act, x + alpha * p, x)
        r = np.where(act, r - alpha * q, r)
        rres = _cnorm(r) / bn_safe
        full = act & (rres <= cfg.tol)
        if full.any():
            tr = _cnorm(b - apply_A(x)) / bn_safe
            rep.matvecs += 1
            ok = full & (tr <= cfg.tol)
            conv |= ok
            iters[ok] = 0.5 * it
        rep.residual_history.append(float(np.max(np.where(act, rres, 0.0))))
        act &= ~conv
        iters[act] = 0.5 * it
        if not act.any():
            break
        z = apply_M(r)
        rep.precond_applications += 1
        rz_new = _cdot(r, z)
        beta = np.where(act, rz_new / np.where(rz != 0, rz, 1.0), 0.0)
        p = np.where(act, z + beta * p, p)
        rz = np.where(act, rz_new, rz)
    rep.col_iterations = iters.tolist()
    rep.iterations = float(iters.max()) if nc else 0.0
    rep.converged = bool(conv.all())
    rep.residual_final = float(np.max(_cnorm(b - apply_A(x)) / bn_safe))
    rep.breakdown = bool(brk.any())
    if brk.any():
        raise BreakdownError("CG breakdown (|p^H A p| or |r^H z| below breakdown_eps)", x, rep)
    return x, rep


def _givens(a, b):
    """Real/complex Givens rotation zeroing b against a: returns (c, s, d)
    with c real, c*a + s*b = d, -conj(s)*a + c*b = 0."""
    if b == 0:
        return 1.0, 0.0 * a, a
    if a == 0:
        return 0.0, np.conj(b) / abs(b), abs(b)
    na, nb = abs(a), abs(b)
    d = math.hypot(na, nb)
    c = na / d
    s = (a / na) * np.conj(b) / d
    return c, s, (a / na) * d


def gmres(apply_A, apply_M, b: np.ndarray, cfg: IterConfig):
    """Right-preconditioned restarted GMRES(m) with CGS2 Arnoldi and Givens
    rotations (new op; not in the reference).

    Columns are independent but batched with aligned cycles: a column leaves
    the cycle when its residual estimate |g_{j+1}|/||b|| <= tol (or it hits
    max_iters); when every active column has left, each updates
    x += Z y (Z = stored preconditioned basis), the true residual
    r = b - A x is recomputed and columns with ||r||/||b|| <= tol are
    converged; the others restart together.  iterations = Arnoldi steps."""
    b = np.asarray(b).reshape(b.shape[0], -1)
    n, nc = b.shape
    m = cfg.restart
    dt = np.result_type(b.dtype, np.float64)
    rep = SolveReport()
    bn = _cnorm(b)
    bn_safe = np.where(bn > 0, bn, 1.0)
    if cfg.initial_guess is not None:
        x = np.array(cfg.initial_guess, dtype=dt).reshape(n, nc)
        r = b - apply_A(x)
        rep.matvecs += 1
    else:
        x = np.zeros((n, nc), dtype=dt)
        r = b.astype(dt, copy=True)
    beta = _cnorm(r)
    conv = (beta / bn_safe <= cfg.tol) | (bn == 0)
    iters = np.zeros(nc, dtype=np.int64)
    rep.residual_history.append(float(np.max(beta / bn_safe)))
    while True:
        act = ~conv & (iters < cfg.max_iters)
        if not act.any():
            break
        V = np.zeros((m + 1, n, nc), dtype=dt)
        Z = np.zeros((m, n, nc), dtype=dt)
        R = np.zeros((m + 1, m, nc), dtype=dt)
        g = np.zeros((m + 1, nc), dtype=dt)
        cs = np.zeros((m, nc))
        sn = np.zeros((m, nc), dtype=dt)
        V[0] = r / np.where(beta > 0, beta, 1.0)
        g[0] = beta
        inner = act.copy()
        steps = np.zeros(nc, dtype=np.int64)
        for j in range(m):
            if not inner.any():
                break
            Z[j] = apply_M(V[j])
            w = apply_A(Z[j])
            rep.precond_applications += 1
            rep.matvecs += 1
            Vj = V[:j + 1]
            h = np.einsum("knc,nc->kc", np.conj(Vj), w)
            w = w - np.einsum("knc,kc->nc", Vj, h)
            h2 = np.einsum("knc,nc->kc", np.conj(Vj), w)
            w = w - np.einsum("knc,kc->nc", Vj, h2)
            h = h + h2
            hn = _cnorm(w)
            V[j + 1] = w / np.where(hn > 0, hn, 1.0)
            hcol = np.zeros((m + 1, nc), dtype=dt)
            hcol[:j + 1] = h
            hcol[j + 1] = hn
            for c in np.flatnonzero(inner):
                for q in range(j):
                    t = cs[q, c] * hcol[q, c] + sn[q, c] * hcol[q + 1, c]
                    hcol[q + 1, c] = -np.conj(sn[q, c]) * hcol[q, c] + cs[q, c] * hcol[q + 1, c]
                    hcol[q, c] = t
                cc, ss, d = _givens(hcol[j, c], hcol[j + 1, c])
                cs[j, c], sn[j, c] = cc, ss
                hcol[j, c], hcol[j + 1, c] = d, 0.0
                g[j + 1, c] = -np.conj(ss) * g[j, c]
                g[j, c] = cc * g[j, c]
                R[:j + 1, j, c] = hcol[:j + 1, c]
                steps[c] += 1
                iters[c] += 1
            est = np.abs(g[j + 1]) / bn_safe
            rep.residual_history.append(float(np.max(np.where(inner, est, 0.0))))
            inner &= (est > cfg.tol) & (iters < cfg.max_iters)
        for c in np.flatnonzero(act):
            kk = int(steps[c])
            if kk == 0:
                continue
            y = sla.solve_triangular(R[:kk, :kk, c], g[:kk, c])
            x[:, c] += np.einsum("knc,k->n", Z[:kk, :, c:c + 1], y)
        r = np.where(act, b - apply_A(x), r)
        rep.matvecs += 1
        beta = np.where(act, _cnorm(r), beta)
        conv |= act & (beta / bn_safe <= cfg.tol)
    rep.col_iterations = iters.astype(float).tolist()
    rep.iterations = float(iters.max()) if nc else 0.0
    rep.converged = bool(conv.all())
    rep.residual_final = float(np.max(_cnorm(b - apply_A(x)) / bn_safe))
    return x, rep


def solve(A: sp.csr_matrix, f: np.ndarray, cfg: SolverConfig, it: IterConfig,
          method: str = "bicgstab", F: SpikeFactorization | None = None):
    """factorize (or reuse F), run the outer Krylov method with
    apply_precond_T (or Block Jacobi) as right preconditioner."""
    A = sp.csr_matrix(A)
    if F is None:
        F = factorize(A, cfg)
    if cfg.variant == "OTF":
        return (*solve_otf(A, F, f, it), F)
    inner0 = F.inner_iterations
    M = {"T": lambda v: apply_precond_T(F, v), "I": lambda v: apply_precond_I(F, v),
         "BJ": lambda v: apply_block_jacobi(F, v)}[cfg.variant]
    Aop = lambda v: A @ v  # noqa: E731
    if method == "bicgstab":
        x, rep = bicgstab(Aop, M, f, it)
    elif method == "gmres":
        x, rep = gmres(Aop, M, f, it)
    elif method == "cg":
        x, rep = cg(Aop, M, f, it)
    else:
        raise ParameterError(method)
    rep.inner_iterations = F.inner_iterations - inner0
    return x, rep, F

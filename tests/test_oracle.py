"""Pin the CPU oracle against every known answer the reference holds for this path.

The reference ships no tests or golden vectors, so
the known answers are the SPEC's per-operation examples ([TRIVIAL]/[DERIVED],
cited per test) and acceptance criteria, plus dense-algebra
identities.  CPU only.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import lrspike_oracle as O


def banded(n, k, seed, dom=4.0, sym=False):
    """Random banded matrix with every diagonal within +-k filled (column and row
    dominance factor ``dom``)."""
    rng = np.random.default_rng(seed)
    diags, offs = [], []
    for d in range(1, k + 1):
        v = rng.uniform(-1, 1, n - d)
        diags += [v, v if sym else rng.uniform(-1, 1, n - d)]
        offs += [d, -d]
    M = sp.diags(diags, offs, shape=(n, n)).tocsr()
    rs = np.maximum(np.abs(M).sum(1).A1, np.abs(M).sum(0).A1)
    return (M + sp.diags(dom * rs + 1.0)).tocsr()


def dense_Sr_truncated(F):
    """Assemble the truncated reduced system S~~_r (2kp x 2kp) densely from the
    low-rank tips (Eq. red_sys_prec_mid_1): per interface [[I, T~_b],[W~_t, I]]."""
    p = F.blocks.layout.p
    k = F.blocks.layout.k
    S = np.eye(2 * k * p)
    for i in range(p - 1):
        sT, sW = F.spT[i], F.spW[i + 1]
        Tb = (sT.u[-k:] * sT.sigma) @ sT.v
        Wt = (sW.u[:k] * sW.sigma) @ sW.v
        bi = slice((2 * i + 1) * k, (2 * i + 2) * k)  # x_{i,b}
        ti = slice((2 * i + 2) * k, (2 * i + 3) * k)  # x_{i+1,t}
        S[bi, ti] = Tb
        S[ti, bi] = Wt
    return S


# ---- partition ------------------------------------------------------------------------
def test_make_layout_examples():
    assert O.make_layout(10, 3, 2).sizes == [4, 3, 3]
    with pytest.raises(O.LayoutError):
        O.make_layout(6, 3, 2)
    assert O.make_layout(1638, 3, 154).sizes == [546, 546, 546]


def test_extract_blocks_examples():
    n = 6
    A = sp.diags([np.full(n - 1, 2.0), np.arange(1.0, 7.0), np.full(n - 1, 3.0)], [-1, 0, 1]).tocsr()
    b = O.extract_blocks(A, O.make_layout(n, 2, 1))
    assert b.B[0].toarray().tolist() == [[3.0]] and b.C[1].toarray().tolist() == [[2.0]]
    D = sp.block_diag([np.ones((3, 3)), 2 * np.ones((3, 3))]).tocsr()
    bd = O.extract_blocks(D, O.make_layout(6, 2, 1))
    assert bd.B[0].nnz == 0 and bd.C[1].nnz == 0
    R = banded(60, 3, 0)
    lay = O.make_layout(60, 4, 3)
    blk = O.extract_blocks(R, lay)  # SPEC.md:188 reassembly
    Z = np.zeros((60, 60))
    for i, (o, s) in enumerate(zip(lay.offsets, lay.sizes)):
        Z[o:o + s, o:o + s] = blk.A[i].toarray()
        if i + 1 < lay.p:
            Z[o + s - 3:o + s, o + s:o + s + 3] = blk.B[i].toarray()
        if i > 0:
            Z[o:o + 3, o - 3:o] = blk.C[i].toarray()
    assert np.array_equal(Z, R.toarray())
    with pytest.raises(O.NotBlockTridiagonalError) as e:
        O.extract_blocks(R, O.make_layout(60, 4, 2))
    assert e.value.row >= 0 and e.value.col >= 0


# ---- block_solver ---------------------------------------------------------------------
def test_block_solver_examples():
    F = O.factorize_block(sp.identity(5, format="csr"))
    assert np.allclose(O.solve_block(F, np.arange(5.0)), np.arange(5.0))
    F2 = O.factorize_block(sp.diags([2.0, 4.0]).tocsr())
    assert np.allclose(O.solve_block(F2, np.array([4.0, 8.0])), [2.0, 2.0])
    R = banded(50, 4, 1)
    F3 = O.factorize_block(R)
    assert np.abs(R.toarray() @ O.solve_block(F3, np.eye(50)) - np.eye(50)).max() <= 1e-11
    Fa = O.factorize_block(sp.csr_matrix([[1.0, 2.0], [0.0, 1.0]]))
    assert np.allclose(O.solve_block_adjoint(Fa, np.array([1.0, 0.0])), [1.0, -2.0])
    S = banded(40, 3, 2, sym=True)
    Fs = O.factorize_block(S)
    r = np.random.default_rng(0).standard_normal(40)
    assert np.allclose(O.solve_block(Fs, r), O.solve_block_adjoint(Fs, r), atol=1e-13)
    with pytest.raises(O.SingularBlockError) as e:
        O.factorize_block(sp.csr_matrix(np.diag([1.0, 0.0, 2.0])))
    assert e.value.column == 1


def test_diagonally_dominant_block_never_swaps():
    # column-diagonally-dominant blocks make no row interchange
    F = O.factorize_block(banded(400, 20, 3, dom=1.0))
    assert F.swaps == 0


# ---- spikes ---------------------------------------------------------------------------
def test_full_spike_examples():
    B = sp.csr_matrix(np.random.default_rng(0).standard_normal((3, 3)))
    FI = O.factorize_block(sp.identity(8, format="csr"))
    T = O.compute_full_spike(FI, B, O.SIDE_T)
    assert np.allclose(T[-3:], B.toarray()) and np.allclose(T[:-3], 0)
    Z = O.compute_full_spike(FI, sp.csr_matrix((3, 3)), O.SIDE_T)
    assert not Z.any()
    R = banded(30, 3, 4)
    FR = O.factorize_block(R)
    T = O.compute_full_spike(FR, B, O.SIDE_T)
    pad = np.zeros((30, 3))
    pad[-3:] = B.toarray()
    assert np.abs(T - np.linalg.solve(R.toarray(), pad)).max() <= 1e-11


def test_randomized_spike_svd_examples():
    R = banded(120, 8, 5)
    FR = O.factorize_block(R)
    rng = np.random.default_rng(1)
    rank1 = sp.csr_matrix(np.outer(rng.standard_normal(8), rng.standard_normal(8)))
    s1 = O.randomized_spike_svd(FR, rank1, O.SIDE_T, 3, 2, 2, 7, 0)
    assert s1.sigma[1] / s1.sigma[0] <= 1e-12
    B = sp.csr_matrix(rng.standard_normal((8, 8)))
    full = O.randomized_spike_svd(FR, B, O.SIDE_W, 8, 0, 4, 7, 0)
    W = O.compute_full_spike(FR, B, O.SIDE_W)
    assert np.linalg.norm(W - (full.u * full.sigma) @ full.v) / np.linalg.norm(W) <= 1e-8
    # orthonormality invariants and fixed-seed reproducibility
    s = O.randomized_spike_svd(FR, B, O.SIDE_T, 4, 2, 2, 11, 0)
    assert np.abs(s.u.T @ s.u - np.eye(4)).max() < 1e-12
    assert np.abs(s.v @ s.v.T - np.eye(4)).max() < 1e-12
    assert np.all(np.diff(s.sigma) <= 0)
    s2 = O.randomized_spike_svd(FR, B, O.SIDE_T, 4, 2, 2, 11, 0)
    assert np.array_equal(s.u, s2.u) and np.array_equal(s.sigma, s2.sigma)
    with pytest.raises(O.ParameterError):
        O.randomized_spike_svd(FR, B, O.SIDE_T, 9, 0, 2, 1, 0)


def test_eckart_young_spike_vs_coupling_svd():
    # acceptance 6: rank-r spike-SVD error <= coupling-SVD-derived error
    viol = 0
    for seed in range(20):
        R = banded(60, 6, 100 + seed, dom=1.5)
        F = O.factorize_block(R)
        B = np.random.default_rng(seed).standard_normal((6, 6))
        T = O.compute_full_spike(F, sp.csr_matrix(B), O.SIDE_T)
        U, s, Vt = np.linalg.svd(T, full_matrices=False)
        Ub, sb, Vbt = np.linalg.svd(B)
        for r in (1, 6 // 4 or 1, 3):
            e_spike = np.linalg.norm(T - (U[:, :r] * s[:r]) @ Vt[:r])
            Br = (Ub[:, :r] * sb[:r]) @ Vbt[:r]
            e_coup = np.linalg.norm(T - O.compute_full_spike(F, sp.csr_matrix(Br), O.SIDE_T))
            viol += e_spike > e_coup + 1e-12
    assert viol == 0


# ---- reduced system / Woodbury ------------------------------------------------------------
def test_woodbury_matches_dense_inverse():
    # acceptance 3: apply_truncated_precond == dense inverse of S~~_r, >= 20 cases
    for seed in range(20):
        k, p = 12, 3
        A = banded(p * 40, k, 200 + seed, dom=1.2)
        F = O.factorize(A, O.SolverConfig(p=p, k=k, n_svd=4, seed=seed))
        rng = np.random.default_rng(seed)
        top = [rng.standard_normal((k, 2)) for _ in range(p)]
        bot = [rng.standard_normal((k, 2)) for _ in range(p)]
        xt, xb = O.apply_truncated_precond(F.trunc, top, bot)
        g = np.concatenate([np.concatenate([t, b]) for t, b in zip(top, bot)])
        x = np.linalg.solve(dense_Sr_truncated(F), g)
        got = np.concatenate([np.concatenate([t, b]) for t, b in zip(xt, xb)])
        assert np.abs(got - x).max() / np.abs(x).max() <= 1e-10


def test_matvec_exact_vs_dense_assembly():
    # p=3 random tips vs dense Eq. 10 assembly
    rng = np.random.default_rng(3)
    k, p = 4, 3
    tipsT = [(rng.standard_normal((k, k)), rng.standard_normal((k, k))) for _ in range(p - 1)]
    tipsW = [None] + [(rng.standard_normal((k, k)), rng.standard_normal((k, k))) for _ in range(p - 1)]
    xt = [rng.standard_normal((k, 1)) for _ in range(p)]
    xb = [rng.standard_normal((k, 1)) for _ in range(p)]
    yt, yb = O.matvec_exact(tipsT, tipsW, xt, xb)
    S = np.eye(2 * k * p)
    for i in range(p):
        r0 = 2 * i * k
        if i > 0:
            S[r0:r0 + k, 2 * (i - 1) * k + k:2 * i * k] = tipsW[i][0]
            S[r0 + k:r0 + 2 * k, 2 * (i - 1) * k + k:2 * i * k] = tipsW[i][1]
        if i < p - 1:
            S[r0:r0 + k, 2 * (i + 1) * k:2 * (i + 1) * k + k] = tipsT[i][0]
            S[r0 + k:r0 + 2 * k, 2 * (i + 1) * k:2 * (i + 1) * k + k] = tipsT[i][1]
    x = np.concatenate([np.concatenate([a, b]) for a, b in zip(xt, xb)])
    y = np.concatenate([np.concatenate([a, b]) for a, b in zip(yt, yb)])
    assert np.abs(S @ x - y).max() <= 1e-14


# ---- spike_solvers ------------------------------------------------------------------------
def test_ds_identity_full_spikes():
    # acceptance 1: D S = A with full spikes
    for p in (2, 3, 4):
        k = 5
        A = banded(p * 50, k, 300 + p)
        lay = O.make_layout(A.shape[0], p, k)
        blk = O.extract_blocks(A, lay)
        D = sp.block_diag(blk.A).toarray()
        S = np.eye(A.shape[0])
        for i, (o, s) in enumerate(zip(lay.offsets, lay.sizes)):
            F = O.factorize_block(blk.A[i])
            if i + 1 < p:
                S[o:o + s, o + s:o + s + k] = O.compute_full_spike(F, blk.B[i], O.SIDE_T)
            if i > 0:
                S[o:o + s, o - k:o] = O.compute_full_spike(F, blk.C[i], O.SIDE_W)
        assert np.linalg.norm(D @ S - A.toarray()) / np.linalg.norm(A.toarray()) <= 1e-12


def test_full_rank_p2_is_exact_solver():
    # SURVEY.md 4 KAT (i): P=2, r=k, exact spike SVD -> LR-SPIKE-T is a direct solver
    A = banded(120, 6, 9, dom=1.0)
    F = O.factorize(A, O.SolverConfig(p=2, k=6, n_svd=6, oversample=0, passes=4, seed=1))
    b = np.random.default_rng(0).standard_normal((120, 2))
    x = O.apply_precond_T(F, b)
    assert np.linalg.norm(x - np.linalg.solve(A.toarray(), b)) / np.linalg.norm(x) <= 1e-12


def test_block_jacobi_limit_bitwise():
    # acceptance 5 + identical outer iterate sequences
    A = banded(160, 6, 10, dom=0.6)
    F = O.factorize(A, O.SolverConfig(p=4, k=6, n_svd=0))
    b = np.random.default_rng(2).standard_normal((160, 1))
    assert np.array_equal(O.apply_precond_T(F, b), O.apply_block_jacobi(F, b))
    it = O.IterConfig(tol=1e-10)
    x1, r1 = O.bicgstab(lambda v: A @ v, lambda v: O.apply_precond_T(F, v), b, it)
    x2, r2 = O.bicgstab(lambda v: A @ v, lambda v: O.apply_block_jacobi(F, v), b, it)
    assert np.array_equal(x1, x2) and r1.residual_history == r2.residual_history


def test_precond_quality_improves_with_rank():
    # SPEC.md:493 / SURVEY.md 4 KAT (iii): residual of A M^-1 f decreases with n_svd
    A = banded(120, 6, 11, dom=0.3)
    f = np.random.default_rng(4).standard_normal((120, 1))
    res = []
    for r in (0, 2, 4, 6):
        F = O.factorize(A, O.SolverConfig(p=4, k=6, n_svd=r, oversample=0, seed=1))
        res.append(np.linalg.norm(A @ O.apply_precond_T(F, f) - f) / np.linalg.norm(f))
    assert res[-1] < res[0] and res[2] < res[0]


def test_ledger_exact_counts():
    # acceptance 9: 4 (p-1) n_svd n_rhs scalars per application
    A = banded(200, 8, 12)
    F = O.factorize(A, O.SolverConfig(p=4, k=8, n_svd=3, seed=2))
    O.apply_precond_T(F, np.ones((200, 2)))
    m1, s1 = F.ledger.stages["precond-apply"]
    m2, s2 = F.ledger.stages["recovery"]
    assert (m1, s1) == (2 * 3, 2 * 3 * 3 * 2) and (m2, s2) == (2 * 3, 2 * 3 * 3 * 2)
    Fb = O.factorize(A, O.SolverConfig(p=4, k=8, n_svd=0))
    O.apply_block_jacobi(Fb, np.ones((200, 1)))
    assert Fb.ledger.stages == {}


def test_block_diagonal_matrix_is_exact():
    # block-diagonal A -> spikes zero, preconditioner exact
    A = sp.block_diag([banded(40, 3, s) for s in range(4)]).tocsr()
    F = O.factorize(A, O.SolverConfig(p=4, k=3, n_svd=2, seed=0))
    b = np.random.default_rng(0).standard_normal((160, 1))
    assert np.allclose(O.apply_precond_T(F, b), np.linalg.solve(A.toarray(), b), atol=1e-12)


# ---- krylov ---------------------------------------------------------------------------------
def test_bicgstab_examples():
    I = sp.identity(10, format="csr")
    b = np.arange(1.0, 11.0)[:, None]
    x, r = O.bicgstab(lambda v: I @ v, lambda v: v, b, O.IterConfig(tol=1e-12))
    assert r.converged and r.iterations == 0.5 and np.allclose(x, b)
    D = sp.diags(np.arange(1.0, 11.0)).tocsr()
    Dinv = sp.diags(1.0 / np.arange(1.0, 11.0)).tocsr()
    x, r = O.bicgstab(lambda v: D @ v, lambda v: Dinv @ v, b, O.IterConfig(tol=1e-12))
    assert r.iterations <= 1 and np.allclose(x, 1.0)
    x, r = O.bicgstab(lambda v: D @ v, lambda v: v, b, O.IterConfig(tol=1e-10))
    assert r.converged and r.iterations <= 10 and np.allclose(x, 1.0, atol=1e-9)
    # precond_applications = 2 x full iterations (+1 trailing half)
    assert r.precond_applications == int(2 * r.iterations)


def test_bicgstab_breakdown_raises_with_partial_result():
    A = sp.csr_matrix(np.array([[0.0, -1.0], [1.0, 0.0]]))  # (t, s) = 0 -> omega = 0
    with pytest.raises(O.BreakdownError) as e:
        O.bicgstab(lambda v: A @ v, lambda v: v, np.array([[1.0], [0.0]]),
                   O.IterConfig(tol=1e-14, max_iters=10, breakdown_eps=1e-30))
    assert e.value.x is not None and e.value.report.breakdown


def test_gmres_matches_direct_solve_and_true_residual():
    A = banded(300, 10, 13, dom=0.2)
    b = np.random.default_rng(5).standard_normal((300, 2))
    x, r = O.gmres(lambda v: A @ v, lambda v: v, b, O.IterConfig(tol=1e-10, restart=20))
    assert r.converged
    assert np.linalg.norm(x - np.linalg.solve(A.toarray(), b)) / np.linalg.norm(x) < 1e-8
    # reported residual == independently recomputed
    rr = np.max(np.linalg.norm(b - A @ x, axis=0) / np.linalg.norm(b, axis=0))
    assert abs(rr - r.residual_final) < 1e-13


def test_multi_rhs_columns_are_independent():
    A = banded(200, 8, 14, dom=0.5)
    F = O.factorize(A, O.SolverConfig(p=4, k=8, n_svd=4, seed=3))
    b = np.random.default_rng(6).standard_normal((200, 3))
    M = lambda v: O.apply_precond_T(F, v)  # noqa: E731
    xb, rb = O.gmres(lambda v: A @ v, M, b, O.IterConfig(tol=1e-9, restart=10))
    for j in range(3):
        xj, rj = O.gmres(lambda v: A @ v, M, b[:, j:j + 1], O.IterConfig(tol=1e-9, restart=10))
        assert rj.col_iterations[0] == rb.col_iterations[j]
        assert np.linalg.norm(xj[:, 0] - xb[:, j]) / np.linalg.norm(xj) < 1e-12

"""Partial pivoting (LAPACK dgbtrf / dgbtrs semantics) for blocks the
no-interchange path rejects: weakly dominant random bands, GPU vs the oracle."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _band(n, k, seed):
    """Row-diagonally-dominant dense band with rows scaled by 10^U[-1.5, 1.5]: well
    conditioned, but a small row's diagonal loses to the large rows below it in its
    column, so dgbtrf interchanges rows in every block."""
    rng = np.random.default_rng(seed)
    offs = [d for d in range(-k, k + 1) if d != 0]
    A = sp.diags([rng.standard_normal(n - abs(d)) for d in offs], offs, shape=(n, n)).tocsr()
    A = (sp.diags(10.0 ** rng.uniform(-1.5, 1.5, n)) @ A).tocsr()
    d = np.asarray(abs(A).sum(axis=1)).ravel() * 1.2 + 1e-3
    return (A + sp.diags(d)).tocsr()


def _gpu(ctx, S):
    return api.CsrMatrix(ctx, S.shape[0], S.indptr, S.indices, S.data)


@pytest.mark.parametrize("n,k,P", [(1200, 40, 3), (4000, 300, 4), (9000, 700, 2)])
def test_pivoted_block_solves_match_lapack(ctx, n, k, P):
    S = _band(n, k, 11)
    lay = O.make_layout(n, P, k)
    blocks = O.extract_blocks(S, lay)
    fos = [O.factorize_block(Ai) for Ai in blocks.A]
    assert all(fo.swaps > 0 for fo in fos)
    F = api.factorize(ctx, _gpu(ctx, S), api.SolverConfig(variant="BJ", p=P, k=k, n_svd=0))
    assert F.info["pivoted"] == 1
    rng = np.random.default_rng(3)
    for i in range(P):
        R = np.asfortranarray(rng.standard_normal((lay.sizes[i], 3)))
        assert _rel(F.solve_block(i, R), O.solve_block(fos[i], R)) < 1e-10
        assert _rel(F.solve_block_adjoint(i, R), O.solve_block_adjoint(fos[i], R)) < 1e-10
        Ad = blocks.A[i].toarray()
        assert _rel(Ad @ F.solve_block(i, R), R) < 1e-9
        X3 = F.solve_block(i, R)
        assert np.array_equal(X3[:, 1], F.solve_block(i, R[:, 1:2])[:, 0])


def test_pivoted_lowrank_solve_parity(ctx):
    n, k, P = 6000, 120, 4
    S = _band(n, k, 5)
    b = np.asfortranarray(np.random.default_rng(1).uniform(-1, 1, (n, 1)))
    gc = api.SolverConfig(variant="T", p=P, k=k, n_svd=16, seed=3)
    oc = O.SolverConfig(variant="T", p=P, k=k, n_svd=16, seed=3)
    A = _gpu(ctx, S)
    F = api.factorize(ctx, A, gc)
    Fo = O.factorize(S, oc)
    assert F.info["pivoted"] == 1
    f = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 2)))
    assert _rel(F.apply_precond_T(f), O.apply_precond_T(Fo, f)) < 1e-9
    it = api.IterConfig(tol=1e-9, method="gmres", restart=40, max_iters=600)
    x, rep, _ = api.solve(A, b, it=it, F=F)
    xo, repo, _ = O.solve(S, b, oc, O.IterConfig(tol=1e-9, restart=40, max_iters=600),
                          method="gmres", F=Fo)
    assert rep.converged and repo.converged
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8


def test_zero_diagonal_needs_interchange(ctx):
    """[[0, 1], [1, 0]] blocks: LAPACK swaps, the result is exact."""
    M = sp.block_diag([sp.csr_matrix(np.array([[0.0, 2.0], [3.0, 1.0]]))] * 4).tocsr()
    A = _gpu(ctx, M)
    F = api.factorize(ctx, A, api.SolverConfig(variant="BJ", p=1, k=1, n_svd=0))
    assert F.info["pivoted"] == 1
    R = np.asfortranarray(np.arange(8.0).reshape(8, 1))
    assert _rel(F.solve_block(0, R), np.linalg.solve(M.toarray(), R)) < 1e-14


def _band_z(n, k, seed):
    """complex128 analogue of _band: random complex band, rows scaled by 10^U[-1.5, 1.5],
    row-dominant diagonal -- zgbtrf (izamax: |Re| + |Im|) interchanges in every block."""
    rng = np.random.default_rng(seed)
    offs = [d for d in range(-k, k + 1) if d != 0]
    A = sp.diags([rng.standard_normal(n - abs(d)) + 1j * rng.standard_normal(n - abs(d))
                  for d in offs], offs, shape=(n, n)).tocsr()
    A = (sp.diags(10.0 ** rng.uniform(-1.5, 1.5, n)) @ A).tocsr()
    d = np.asarray(abs(A).sum(axis=1)).ravel() * 1.2 + 1e-3
    ph = np.exp(1j * rng.uniform(0, 2 * np.pi, n))
    return (A + sp.diags(d * ph)).tocsr()


@pytest.mark.parametrize("n,k,P", [(1200, 40, 3), (4000, 300, 4)])
def test_pivoted_complex_block_solves_match_lapack(ctx, n, k, P):
    S = _band_z(n, k, 13)
    lay = O.make_layout(n, P, k)
    blocks = O.extract_blocks(S, lay)
    fos = [O.factorize_block(Ai) for Ai in blocks.A]
    assert all(fo.swaps > 0 for fo in fos)
    F = api.factorize(ctx, _gpu(ctx, S), api.SolverConfig(variant="BJ", p=P, k=k, n_svd=0))
    assert F.info["pivoted"] == 1
    rng = np.random.default_rng(4)
    for i in range(P):
        R = np.asfortranarray(rng.standard_normal((lay.sizes[i], 3))
                              + 1j * rng.standard_normal((lay.sizes[i], 3)))
        X = F.solve_block(i, R)
        assert _rel(X, O.solve_block(fos[i], R)) < 1e-10
        assert _rel(F.solve_block_adjoint(i, R), O.solve_block_adjoint(fos[i], R)) < 1e-10
        Ad = blocks.A[i].toarray()
        assert _rel(Ad @ X, R) < 1e-9
        assert _rel(Ad.conj().T @ F.solve_block_adjoint(i, R), R) < 1e-9
        assert np.array_equal(X[:, 2], F.solve_block(i, R[:, 2:3])[:, 0])


def test_pivoted_complex_lowrank_solve_parity(ctx):
    n, k, P = 5000, 100, 4
    S = _band_z(n, k, 7)
    rng = np.random.default_rng(1)
    b = np.asfortranarray(rng.uniform(-1, 1, (n, 2)) + 1j * rng.uniform(-1, 1, (n, 2)))
    gc = api.SolverConfig(variant="T", p=P, k=k, n_svd=16, seed=3)
    oc = O.SolverConfig(variant="T", p=P, k=k, n_svd=16, seed=3)
    A = _gpu(ctx, S)
    F = api.factorize(ctx, A, gc)
    Fo = O.factorize(S, oc)
    assert F.info["pivoted"] == 1
    f = np.asfortranarray(rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2)))
    assert _rel(F.apply_precond_T(f), O.apply_precond_T(Fo, f)) < 1e-9
    it = api.IterConfig(tol=1e-9, method="gmres", restart=40, max_iters=600)
    x, rep, _ = api.solve(A, b, it=it, F=F)
    xo, repo, _ = O.solve(S, b, oc, O.IterConfig(tol=1e-9, restart=40, max_iters=600),
                          method="gmres", F=Fo)
    assert rep.converged and repo.converged
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8


def test_symmetric_block_that_interchanges_leaves_the_symmetric_schedule(ctx):
    """A symmetric band whose blocks need row interchanges (a dominant symmetric band with a
    few diagonal entries shrunk to 1e-6): the symmetric no-interchange schedule starts
    (A == A^T, band of >= 3 tiles), its pivot test fires on the L panel, and the blocks are
    redone on the partial-pivoting path -- fact_info reports pivoted, not lu_sym; block solves
    equal LAPACK's."""
    n, k, P = 6000, 520, 2
    rng = np.random.default_rng(21)
    offs = list(range(1, k + 1))
    up = sp.diags([rng.standard_normal(n - d) for d in offs], offs, shape=(n, n)).tocsr()
    A = (up + up.T).tocsr()
    d = np.asarray(abs(A).sum(axis=1)).ravel() * 1.2 + 1e-3
    weak = rng.choice(n, size=12, replace=False)
    d[weak] = 1e-6
    S = (A + sp.diags(d)).tocsr()
    S.sort_indices()
    assert abs(S - S.T).max() == 0.0
    lay = O.make_layout(n, P, k)
    blocks = O.extract_blocks(S, lay)
    fos = [O.factorize_block(Ai) for Ai in blocks.A]
    assert any(fo.swaps > 0 for fo in fos)
    F = api.factorize(ctx, _gpu(ctx, S), api.SolverConfig(variant="BJ", p=P, k=k, n_svd=0))
    assert F.info["pivoted"] == 1 and F.info["lu_sym"] == 0
    R = np.asfortranarray(rng.standard_normal((lay.sizes[0], 2)))
    for i in range(P):
        R = np.asfortranarray(rng.standard_normal((lay.sizes[i], 2)))
        assert _rel(F.solve_block(i, R), O.solve_block(fos[i], R)) < 1e-8
        assert _rel(blocks.A[i].toarray() @ F.solve_block(i, R), R) < 1e-8

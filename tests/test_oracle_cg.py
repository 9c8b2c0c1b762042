"""The checker's preconditioned CG (SPEC.md:430-436 examples).  CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import lrspike_oracle as O


def _lap2d(g):
    T = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(g, g))
    return (sp.kron(sp.eye(g), T) + sp.kron(T, sp.eye(g))).tocsr()


def test_cg_identity_half_iteration():
    b = np.arange(1.0, 6.0).reshape(5, 1)
    x, rep = O.cg(lambda v: v, lambda v: v, b, O.IterConfig(tol=1e-12))
    assert rep.iterations == 0.5 and rep.converged
    assert np.array_equal(x, b)


def test_cg_laplacian_matches_dense():
    A = _lap2d(16)
    b = np.random.default_rng(0).standard_normal((A.shape[0], 3))
    x, rep = O.cg(lambda v: A @ v, lambda v: v, b, O.IterConfig(tol=1e-12, max_iters=500))
    assert rep.converged
    xd = np.linalg.solve(A.toarray(), b)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-10
    assert abs(rep.residual_final - np.max(np.linalg.norm(A @ x - b, axis=0) /
                                           np.linalg.norm(b, axis=0))) < 1e-13


def test_cg_block_jacobi_preconditioner_reduces_iterations():
    A = _lap2d(24) + 1e-2 * sp.eye(576)
    A = A.tocsr()
    b = np.ones((A.shape[0], 1))
    F = O.factorize(A, O.SolverConfig(variant="BJ", p=4, k=24, n_svd=0))
    it = O.IterConfig(tol=1e-10, max_iters=1000)
    _, r0 = O.cg(lambda v: A @ v, lambda v: v, b, it)
    x, r1 = O.cg(lambda v: A @ v, lambda v: O.apply_block_jacobi(F, v), b, it)
    assert r0.converged and r1.converged and r1.iterations < r0.iterations
    assert r1.precond_applications == 2 * r1.iterations or r1.precond_applications == 2 * r1.iterations + 1


def test_cg_indefinite_breaks_down():
    A = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]]))
    b = np.array([[1.0], [0.0]])
    with pytest.raises(O.BreakdownError) as e:
        O.cg(lambda v: A @ v, lambda v: v, b, O.IterConfig(tol=1e-12, max_iters=10))
    assert e.value.report.breakdown

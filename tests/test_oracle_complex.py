"""The checker's complex128 path (config c5): the shifted FEAST systems, the
conjugate-transpose adjoint and the Hermitian range finder.  CPU only."""
import numpy as np
import scipy.sparse as sp

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import configs


def test_shifted_system_is_zI_minus_A():
    cfg = configs.make_config("c5", 8 / 80, P=2)
    A = cfg.matrix.to_scipy()
    z = cfg.shifts[3]
    Z = cfg.system(3).to_scipy()
    assert Z.dtype == np.complex128
    assert abs(Z - (z * sp.identity(A.shape[0]) - A)).max() == 0
    assert len(cfg.shifts) == 8
    assert all(abs(abs(s - 2.0) - 0.5) < 1e-15 for s in cfg.shifts)


def test_complex_adjoint_is_conjugate_transpose():
    rng = np.random.default_rng(0)
    n = 40
    M = np.diag(4 + 1j * rng.uniform(-1, 1, n))
    for d in (1, 2):
        M += np.diag(rng.uniform(-1, 1, n - d) + 1j * rng.uniform(-1, 1, n - d), d)
        M += np.diag(rng.uniform(-1, 1, n - d) + 1j * rng.uniform(-1, 1, n - d), -d)
    F = O.factorize_block(sp.csr_matrix(M))
    R = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
    assert np.allclose(O.solve_block(F, R), np.linalg.solve(M, R), rtol=1e-12, atol=1e-13)
    assert np.allclose(O.solve_block_adjoint(F, R), np.linalg.solve(M.conj().T, R),
                       rtol=1e-12, atol=1e-13)


def test_complex_spike_svd_captures_the_spike():
    """rank-r approximation of the exact spike T = A_i^-1 [0; B_i] is near-optimal:
    ||T - u S v|| close to sigma_{r+1}(T) (Hermitian form)."""
    cfg = configs.make_config("c5", 10 / 80, P=2)
    A = cfg.system(1).to_scipy()
    lay = O.make_layout(A.shape[0], 2, cfg.b)
    bl = O.extract_blocks(A, lay)
    F = O.factorize_block(bl.A[0])
    r = 8
    s = O.randomized_spike_svd(F, bl.B[0], O.SIDE_T, r, 8, 4, cfg.seed, 0)
    T = O.compute_full_spike(F, bl.B[0], O.SIDE_T)
    sv = np.linalg.svd(T, compute_uv=False)
    err = np.linalg.norm(T - (s.u * s.sigma) @ s.v, 2)
    assert err <= 10 * sv[r]
    # Rayleigh-Ritz values: below the true singular values, and close to them
    assert np.all(s.sigma <= sv[:r] * (1 + 1e-12))
    assert np.all(s.sigma >= 0.9 * sv[:r])
    # orthonormal factors
    assert np.allclose(s.u.conj().T @ s.u, np.eye(r), atol=1e-12)
    assert np.allclose(s.v @ s.v.conj().T, np.eye(r), atol=1e-12)

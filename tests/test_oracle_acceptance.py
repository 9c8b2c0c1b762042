"""SPEC acceptance criteria 8 and 10 on the CPU oracle."""
import numpy as np

from oracle import lrspike_oracle as O
from tests.acceptance_cases import ACC8_RANKS, banded, cond2, convection_diffusion_2d


def test_acceptance8_condition_number_trend():
    """cond(M^-1 A) of LR-SPIKE-T at p = 3 strictly decreases over n_svd in {0, 4, 8, 16},
    and at n_svd >= 8 is <= 1/5 of Block Jacobi's (n_svd = 0)."""
    A = convection_diffusion_2d()
    Ad = np.asfortranarray(A.toarray())
    cs = []
    for r in ACC8_RANKS:
        F = O.factorize(A, O.SolverConfig(p=3, k=42, n_svd=r, seed=0))
        cs.append(cond2(O.apply_precond_T(F, Ad)))
    assert all(b < a for a, b in zip(cs, cs[1:])), cs
    assert cs[2] <= cs[0] / 5 and cs[3] <= cs[0] / 5, cs


def test_acceptance10_dominance_decay():
    """||T_{i,t}||_F / ||T_{i,b}||_F decreases as the dominance factor grows, and
    LR-SPIKE-T with n_svd = 4 reaches 1e-10 in <= 5 outer iterations at d = 4."""
    for seed in (0, 1, 2):
        ratios = []
        for d in (1.5, 2.0, 4.0):
            A = banded(96, 8, 40 + seed, dom=d)
            blk = O.extract_blocks(A, O.make_layout(96, 3, 8))
            T = O.compute_full_spike(O.factorize_block(blk.A[0]), blk.B[0], O.SIDE_T)
            ratios.append(np.linalg.norm(T[:8]) / np.linalg.norm(T[-8:]))
        assert ratios[0] > ratios[1] > ratios[2], ratios
        A = banded(600, 8, 40 + seed, dom=4.0)
        b = np.random.default_rng(1).standard_normal((600, 1))
        _, rep, _ = O.solve(A, b, O.SolverConfig(p=3, k=8, n_svd=4, seed=0),
                            O.IterConfig(tol=1e-10))
        assert rep.converged and rep.iterations <= 5

"""SPEC acceptance criteria 8 and 10 on the GPU solver, against the
same properties and the oracle's numbers."""
import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api
from tests.acceptance_cases import ACC8_RANKS, banded, cond2, convection_diffusion_2d, to_csr

pytestmark = pytest.mark.gpu


def test_acceptance8_condition_number_trend_gpu(ctx):
    A = convection_diffusion_2d()
    Ag = api.CsrMatrix.from_csr(ctx, to_csr(A))
    Ad = np.asfortranarray(A.toarray())
    cs, co = [], []
    for r in ACC8_RANKS:
        F = api.factorize(ctx, Ag, api.SolverConfig(p=3, k=42, n_svd=r, seed=0))
        cs.append(cond2(F.apply_precond_T(Ad)))
        Fo = O.factorize(A, O.SolverConfig(p=3, k=42, n_svd=r, seed=0))
        co.append(cond2(O.apply_precond_T(Fo, Ad)))
        del F
    assert all(b < a for a, b in zip(cs, cs[1:])), cs
    assert cs[2] <= cs[0] / 5 and cs[3] <= cs[0] / 5, cs
    assert np.allclose(cs, co, rtol=1e-8), (cs, co)


def test_acceptance10_dominance_decay_gpu(ctx):
    for seed in (0, 1, 2):
        ratios = []
        for d in (1.5, 2.0, 4.0):
            A = banded(96, 8, 40 + seed, dom=d)
            # full rank (n_svd = k, no oversampling): the low-rank spike is the spike
            F = api.factorize(ctx, api.CsrMatrix.from_csr(ctx, to_csr(A)),
                              api.SolverConfig(p=3, k=8, n_svd=8, oversample=0, seed=0))
            u, s, v = F.spike(0, api.SIDE_T)
            T = (u * s) @ v
            ratios.append(np.linalg.norm(T[:8]) / np.linalg.norm(T[-8:]))
            del F
        assert ratios[0] > ratios[1] > ratios[2], ratios
        A = banded(600, 8, 40 + seed, dom=4.0)
        b = np.random.default_rng(1).standard_normal((600, 1))
        x, rep, _ = api.solve(api.CsrMatrix.from_csr(ctx, to_csr(A)), b,
                              api.SolverConfig(p=3, k=8, n_svd=4, seed=0),
                              api.IterConfig(tol=1e-10, method="bicgstab"))
        assert rep.converged and rep.iterations <= 5
        assert rep.residual_final <= 1e-10

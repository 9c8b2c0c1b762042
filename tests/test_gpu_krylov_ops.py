"""bicgstab / cg / GMRES on caller-supplied operators (the Krylov
drivers take abstract operator and preconditioner contracts), through lrs_krylov."""
import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().t()


@pytest.mark.parametrize("method", ["bicgstab", "cg", "gmres"])
def test_krylov_on_caller_operators(ctx, method):
    cfg = configs.make_config("c1", 48 / 256)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    F = api.factorize(ctx, A, api.SolverConfig(variant="BJ", p=cfg.P, k=cfg.b, n_svd=0))
    Fo = O.factorize(S, O.SolverConfig(variant="BJ", p=cfg.P, k=cfg.b, n_svd=0))
    b = np.asfortranarray(np.random.default_rng(4).uniform(-1, 1, (S.shape[0], 2)))
    it = api.IterConfig(tol=1e-9, method=method, restart=30, max_iters=600)
    x, rep = api.krylov(ctx, lambda u, v: A.spmv(u, v), _dev(b), it,
                        apply_M=lambda u, v: F.apply_block_jacobi(u, v))
    oit = O.IterConfig(tol=1e-9, restart=30, max_iters=600)
    fn = {"bicgstab": O.bicgstab, "cg": O.cg, "gmres": O.gmres}[method]
    xo, repo = fn(lambda v: S @ v, lambda v: O.apply_block_jacobi(Fo, v), b, oit)
    assert rep.converged and repo.converged
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x.cpu().numpy(), xo) <= 1e-8
    assert rep.residual_final <= 1e-9


def test_krylov_identity_and_host_buffers(ctx):
    b = np.asfortranarray(np.arange(1.0, 11.0).reshape(10, 1))
    x, rep = api.krylov(ctx, lambda u, v: v.copy_(u), b, api.IterConfig(tol=1e-12))
    assert rep.iterations == 0.5 and np.array_equal(x, b)
    x, rep = api.krylov(ctx, lambda u, v: v.copy_(u), b, api.IterConfig(tol=1e-12, method="cg"))
    assert rep.iterations == 0.5 and np.allclose(x, b)


def test_krylov_callback_failure_is_reported(ctx):
    def bad(u, v):
        raise RuntimeError("operator failed")

    with pytest.raises(api.Error):
        api.krylov(ctx, bad, np.ones((8, 1), order="F"), api.IterConfig(tol=1e-10))

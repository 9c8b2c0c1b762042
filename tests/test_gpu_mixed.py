"""Mixed precision: FP32 off-diagonal factor tiles
in the preconditioner applies, FP64 everywhere else.  The oracle emulates it exactly
(round_offdiag_tiles), so the usual parity bars apply."""
import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name,scale,method", [("c2", 16 / 64, "bicgstab"), ("c1", 64 / 256, "gmres")])
def test_fp32_factors_parity(ctx, name, scale, method):
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    gc = api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed, factor_fp32=True)
    oc = O.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed,
                        factor_fp32=True)
    F = api.factorize(ctx, A, gc)
    Fo = O.factorize(S, oc)
    F64 = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
    assert F.info["factor_bytes"] > F64.info["factor_bytes"]
    assert F.info["apply_bytes"] <= F64.info["apply_bytes"]
    if cfg.b >= 1024:  # wide bands: the FP32 off-diagonal tiles dominate the factor stream
        assert F.info["apply_bytes"] < 0.7 * F64.info["apply_bytes"]
    f = np.asfortranarray(np.random.default_rng(8).uniform(-1, 1, (S.shape[0], 2)))
    y = F.apply_precond_T(f)
    assert _rel(y, O.apply_precond_T(Fo, f)) < 1e-10
    assert _rel(F.apply_block_jacobi(f), O.apply_block_jacobi(Fo, f)) < 1e-10
    assert 1e-12 < _rel(y, F64.apply_precond_T(f)) < 1e-5  # FP32 rounding, not FP64
    # the one-column apply runs the FMA sweeps (four partial sums per FP32 chunk)
    f1 = np.asfortranarray(f[:, :1])
    assert _rel(F.apply_precond_T(f1), O.apply_precond_T(Fo, f1)) < 1e-10
    # the FP32 copy holds only the tile slots inside their block: at most half the FP64 bytes
    assert F.info["factor_bytes"] - F64.info["factor_bytes"] <= F64.info["factor_bytes"] // 2
    it = api.IterConfig(tol=cfg.tol, method=method, restart=cfg.m or 30, max_iters=500)
    x, rep, _ = api.solve(A, cfg.rhs, it=it, F=F)
    xo, repo, _ = O.solve(S, cfg.rhs, oc, O.IterConfig(tol=cfg.tol, restart=cfg.m or 30,
                                                       max_iters=500), method=method, F=Fo)
    assert rep.converged and repo.converged and rep.residual_final <= cfg.tol
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8

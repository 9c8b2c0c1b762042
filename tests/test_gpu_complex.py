"""complex128 parity (config c5): the FEAST contour systems
z_j I - A through the CUDA path, against the CPU oracle (zgbtrf / zgbtrs, the
conjugate-transpose range finder, Hermitian Krylov dots, complex Givens).

Tolerances as in test_gpu_parity.py: kernel-level 1e-12 (block solves) / 1e-10
(preconditioner apply), end to end solution relative difference <= 1e-8, true
residual <= tol, iterations within 2.
"""
import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _crand(rng, shape):
    return np.asfortranarray(rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape))


def _c5(scale=16 / 80, P=4, shift=0):
    cfg = configs.make_config("c5", scale, P=P)
    return cfg, cfg.system(shift)


@pytest.mark.parametrize("shift", [0, 5])
def test_complex_spmv(ctx, shift):
    cfg, Az = _c5(shift=shift)
    A = api.CsrMatrix.from_csr(ctx, Az)
    assert A.dtype == np.complex128
    X = _crand(np.random.default_rng(0), (Az.n, 3))
    assert _rel(A.spmv(X), Az.to_scipy() @ X) < 1e-14


@pytest.mark.parametrize("shift", [0, 3])
def test_complex_solve_block_and_adjoint(ctx, shift):
    cfg, Az = _c5(shift=shift)
    S = Az.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, Az)
    F = api.factorize(ctx, A, api.SolverConfig(variant="BJ", p=cfg.P, k=cfg.b, n_svd=0))
    lay = O.make_layout(S.shape[0], cfg.P, cfg.b)
    blocks = O.extract_blocks(S, lay)
    rng = np.random.default_rng(11)
    for i in range(cfg.P):
        fo = O.factorize_block(blocks.A[i])
        assert fo.swaps == 0
        R = _crand(rng, (lay.sizes[i], 3))
        assert _rel(F.solve_block(i, R), O.solve_block(fo, R)) < 1e-12
        # adjoint = conjugate transpose A_i^-H
        Xa = F.solve_block_adjoint(i, R)
        assert _rel(Xa, O.solve_block_adjoint(fo, R)) < 1e-12
        Ad = blocks.A[i].toarray()
        assert _rel(Ad.conj().T @ Xa, R) < 1e-10
        X3 = F.solve_block(i, R)
        X1 = F.solve_block(i, R[:, 1:2])
        assert np.array_equal(X3[:, 1], X1[:, 0])


@pytest.mark.parametrize("shift,r", [(0, 8), (6, 16)])
def test_complex_apply_precond_matches_oracle(ctx, shift, r):
    cfg, Az = _c5(shift=shift)
    S = Az.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, Az)
    F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=r, seed=cfg.seed))
    Fo = O.factorize(S, O.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=r, seed=cfg.seed))
    assert F.n_svd == Fo.n_svd
    f = _crand(np.random.default_rng(4), (S.shape[0], 5))
    assert _rel(F.apply_precond_T(f), O.apply_precond_T(Fo, f)) < 1e-10
    assert _rel(F.apply_block_jacobi(f), O.apply_block_jacobi(Fo, f)) < 1e-12
    for i, side in ((0, api.SIDE_T), (1, api.SIDE_W)):
        u, s, v = F.spike(i, side)
        so = Fo.spT[i] if side == api.SIDE_T else Fo.spW[i]
        assert _rel(s, so.sigma) < 1e-10
        assert _rel((u * s) @ v, (so.u * so.sigma) @ so.v) < 1e-9


@pytest.mark.parametrize("shift,nrhs", [(0, 16), (4, 3)])
def test_complex_gmres_parity(ctx, shift, nrhs):
    cfg, Az = _c5(shift=shift)
    S = Az.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, Az)
    b = np.asfortranarray(cfg.rhs[:, :nrhs].astype(np.complex128))
    it = api.IterConfig(tol=cfg.tol, method="gmres", restart=cfg.m, max_iters=600)
    scfg = api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    x, rep, F = api.solve(A, b, scfg, it)
    xo, repo, _ = O.solve(S, b, O.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=cfg.r,
                                                seed=cfg.seed),
                          O.IterConfig(tol=cfg.tol, restart=cfg.m, max_iters=600), method="gmres")
    assert rep.converged and repo.converged
    assert rep.residual_final <= cfg.tol
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8
    assert _rel(S @ x, b) <= 10 * cfg.tol


def test_complex_bicgstab_parity(ctx):
    cfg, Az = _c5(shift=2)
    S = Az.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, Az)
    b = np.asfortranarray(cfg.rhs[:, :2].astype(np.complex128))
    it = api.IterConfig(tol=1e-9, method="bicgstab", max_iters=600)
    x, rep, F = api.solve(A, b, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=16, seed=cfg.seed), it)
    xo, repo, _ = O.solve(S, b, O.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=16,
                                                seed=cfg.seed),
                          O.IterConfig(tol=1e-9, max_iters=600), method="bicgstab")
    assert rep.converged and repo.converged
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8


def test_complex_device_buffers(ctx):
    import torch

    cfg, Az = _c5(shift=1)
    A = api.CsrMatrix.from_csr(ctx, Az)
    F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=8, seed=cfg.seed))
    f = _crand(np.random.default_rng(9), (Az.n, 2))
    torch.cuda.synchronize()
    fd = torch.from_numpy(np.ascontiguousarray(f.T)).cuda().t()
    torch.cuda.synchronize()
    xd = F.apply_precond_T(fd)
    ctx.synchronize()
    assert _rel(xd.cpu().numpy(), F.apply_precond_T(f)) == 0.0

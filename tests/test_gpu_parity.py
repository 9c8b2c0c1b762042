"""GPU parity tests: the CUDA path (through the C-ABI) against the CPU oracle on
identical seeded inputs.  Run on a B200 with ``pytest -m gpu``.

Tolerances (north_star): solution relative difference <= 1e-8, final true
relative residual <= tol, iteration count within 2 of the oracle.  Kernel-level
parity (block factors, block solves, preconditioner applies) is checked at
1e-12 relative, well inside the FP64 roundoff of the different summation orders.
"""
import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _oracle_cfg(cfg, r, variant="T"):
    return O.SolverConfig(variant=variant, p=cfg.P, k=cfg.b, n_svd=r, seed=cfg.seed)


def _gpu_cfg(cfg, r, variant="T"):
    return api.SolverConfig(variant=variant, p=cfg.P, k=cfg.b, n_svd=r, seed=cfg.seed)


def test_dmma_peak_positive(ctx):
    tf = ctx.dmma_peak_tflops()
    assert 1.0 < tf < 200.0


@pytest.mark.parametrize("name,scale", [("c1", 48 / 256), ("c1", 128 / 256), ("c2", 16 / 64),
                                        ("c2", 24 / 64)])
def test_block_factors_match_lapack(ctx, name, scale):
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    F = api.factorize(ctx, A, _gpu_cfg(cfg, 0, "BJ"))
    lay = O.make_layout(S.shape[0], cfg.P, cfg.b)
    blocks = O.extract_blocks(S, lay)
    nb, wl = F.info["nb"], F.info["wl"]
    for i in (0, cfg.P - 1):
        fo = O.factorize_block(blocks.A[i], F.info["kl"], F.info["ku"])
        assert fo.swaps == 0
        n_i = lay.sizes[i]
        # dense LAPACK L (unit lower) and U
        Lr = np.eye(n_i)
        Ur = np.zeros((n_i, n_i))
        kl, ku = fo.kl, fo.ku
        for j in range(n_i):
            for q in range(max(0, j - ku - kl), min(n_i, j + kl + 1)):
                v = fo.ab[kl + ku + q - j, j]
                if q > j:
                    Lr[q, j] = v
                else:
                    Ur[q, j] = v
        tl = F.tiles(i)
        T = tl.shape[0]
        Lg = np.eye(T * nb)
        Ug = np.zeros((T * nb, T * nb))
        W = tl.shape[1]
        for I in range(T):
            for s in range(W):
                J = I + s - wl
                if J < 0 or J >= T:
                    continue
                blk = tl[I, s]
                if J < I:
                    Lg[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb] = blk
                elif J > I:
                    Ug[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb] = blk
                else:
                    iL = np.tril(blk, -1) + np.eye(nb)
                    iU = np.triu(blk)
                    Lg[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb] = np.linalg.inv(iL)
                    Ug[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb] = np.linalg.inv(iU)
        assert _rel(Lg[:n_i, :n_i], Lr) < 1e-12
        assert _rel(Ug[:n_i, :n_i], Ur) < 1e-12


@pytest.mark.parametrize("name,scale", [("c1", 48 / 256), ("c2", 24 / 64)])
def test_solve_block_and_adjoint(ctx, name, scale):
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    F = api.factorize(ctx, A, _gpu_cfg(cfg, 0, "BJ"))
    lay = O.make_layout(S.shape[0], cfg.P, cfg.b)
    blocks = O.extract_blocks(S, lay)
    rng = np.random.default_rng(7)
    for i in range(cfg.P):
        fo = O.factorize_block(blocks.A[i])
        R = np.asfortranarray(rng.standard_normal((lay.sizes[i], 3)))
        assert _rel(F.solve_block(i, R), O.solve_block(fo, R)) < 1e-12
        assert _rel(F.solve_block_adjoint(i, R), O.solve_block_adjoint(fo, R)) < 1e-12
        # multi-column equals column-by-column bit-exactly
        X3 = F.solve_block(i, R)
        X1 = F.solve_block(i, R[:, 1:2])
        assert np.array_equal(X3[:, 1], X1[:, 0])


@pytest.mark.parametrize("name,scale,r", [("c1", 48 / 256, 8), ("c2", 16 / 64, 16),
                                          ("c2", 24 / 64, 16)])
def test_apply_precond_matches_oracle(ctx, name, scale, r):
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    F = api.factorize(ctx, A, _gpu_cfg(cfg, r))
    Fo = O.factorize(S, _oracle_cfg(cfg, r))
    assert F.n_svd == Fo.n_svd
    f = np.asfortranarray(np.random.default_rng(3).uniform(-1, 1, (S.shape[0], 2)))
    xg = F.apply_precond_T(f)
    xo = O.apply_precond_T(Fo, f)
    assert _rel(xg, xo) < 1e-10
    bj_g = F.apply_block_jacobi(f)
    assert _rel(bj_g, O.apply_block_jacobi(Fo, f)) < 1e-12
    # spikes: the rank-r operator u S v is basis independent
    for i, side in ((0, api.SIDE_T), (1, api.SIDE_W)):
        u, s, v = F.spike(i, side)
        so = Fo.spT[i] if side == api.SIDE_T else Fo.spW[i]
        assert _rel(s, so.sigma) < 1e-10
        assert _rel((u * s) @ v, (so.u * so.sigma) @ so.v) < 1e-9


def test_r0_equals_block_jacobi_bitwise(ctx):
    cfg = configs.make_config("c1", 48 / 256)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    F = api.factorize(ctx, A, _gpu_cfg(cfg, 0, "T"))
    f = np.asfortranarray(np.random.default_rng(1).uniform(-1, 1, (cfg.matrix.n, 1)))
    assert np.array_equal(F.apply_precond_T(f), F.apply_block_jacobi(f))


@pytest.mark.parametrize("name,scale,method", [("c1", 48 / 256, "gmres"), ("c1", 96 / 256, "gmres"),
                                               ("c2", 16 / 64, "bicgstab"),
                                               ("c2", 24 / 64, "bicgstab"),
                                               ("c1", 48 / 256, "bicgstab")])
def test_solve_parity(ctx, name, scale, method):
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    it = api.IterConfig(tol=cfg.tol, method=method, restart=cfg.m or 30, max_iters=500)
    x, rep, F = api.solve(A, cfg.rhs, _gpu_cfg(cfg, cfg.r), it)
    xo, repo, _ = O.solve(S, cfg.rhs, _oracle_cfg(cfg, cfg.r),
                          O.IterConfig(tol=cfg.tol, restart=cfg.m or 30, max_iters=500),
                          method=method)
    assert rep.converged and repo.converged
    assert rep.residual_final <= cfg.tol
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8
    # ledger: 4 (p-1) n_svd n_rhs scalars per application
    m, s = rep.comm["precond-apply"]
    assert s == 2 * (cfg.P - 1) * F.n_svd * rep.precond_applications


@pytest.mark.parametrize("key", ["c1_s48", "c2_s16"])
def test_gpu_matches_golden_fixtures(ctx, key):
    import json
    import os

    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    case = json.load(open(os.path.join(gold, "golden.json")))["cases"][key]
    z = np.load(os.path.join(gold, f"{key}.npz"))
    cfg = configs.make_config(case["config"], case["scale"])
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    it = api.IterConfig(tol=cfg.tol, method=case["method"], restart=cfg.m or 30)
    x, rep, F = api.solve(A, cfg.rhs, _gpu_cfg(cfg, cfg.r), it)
    assert abs(rep.iterations - case["iterations"]) <= 2
    assert _rel(x, z["x"]) <= 1e-8
    assert _rel(F.apply_precond_T(np.asfortranarray(z["apply_in"])), z["apply_out"]) <= 1e-10


def test_cpp_api_on_gpu():
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_api")
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_device_resident_torch_buffers(ctx):
    import torch

    cfg = configs.make_config("c2", 16 / 64)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    F = api.factorize(ctx, A, _gpu_cfg(cfg, cfg.r))
    f = np.asfortranarray(np.random.default_rng(5).uniform(-1, 1, (cfg.matrix.n, 3)))
    torch.cuda.synchronize()
    fd = torch.from_numpy(f.T.copy()).cuda().t()  # column-major on the device
    torch.cuda.synchronize()
    xd = F.apply_precond_T(fd)
    ctx.synchronize()
    assert _rel(xd.cpu().numpy(), F.apply_precond_T(f)) == 0.0
    y = A.spmv(fd)
    ctx.synchronize()
    assert _rel(y.cpu().numpy(), cfg.matrix.to_scipy() @ f) < 1e-14


def test_error_paths(ctx):
    cfg = configs.make_config("c1", 48 / 256)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    with pytest.raises(api.LayoutError):
        api.factorize(ctx, A, api.SolverConfig(p=100, k=48, n_svd=4))
    with pytest.raises(api.NotBlockTridiagonalError) as e:
        api.factorize(ctx, A, api.SolverConfig(p=4, k=20, n_svd=4))
    assert e.value.row >= 0 and e.value.col >= 0
    with pytest.raises(api.ParameterError):
        api.factorize(ctx, A, api.SolverConfig(p=4, k=48, n_svd=47))
    with pytest.raises(api.DimensionError):
        api.CsrMatrix(ctx, 3, [0, 2, 2, 3], [1, 0, 1], [1.0, 1.0, 1.0])  # decreasing cols
    # zero pivot -> SingularBlockError(column)
    import scipy.sparse as sp

    Z = sp.csr_matrix(np.diag([1.0, 0.0, 2.0, 3.0]))
    Az = api.CsrMatrix(ctx, 4, Z.indptr, Z.indices, Z.data)
    with pytest.raises(api.SingularBlockError) as es:
        api.factorize(ctx, Az, api.SolverConfig(variant="BJ", p=1, k=0, n_svd=0))
    assert es.value.column == 1


@pytest.mark.parametrize("name,scale", [("c1", 64 / 256), ("c3", 12 / 96)])
def test_cg_parity(ctx, name, scale):
    """PCG on the SPD c1 / c3 systems with the Block Jacobi
    preconditioner (symmetric for symmetric A; the LR-SPIKE-T preconditioner is not,
    and PCG does not converge with it): GPU vs oracle."""
    variant, r = "BJ", 0
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    it = api.IterConfig(tol=1e-9, method="cg", max_iters=800)
    x, rep, F = api.solve(A, cfg.rhs, _gpu_cfg(cfg, r, variant), it)
    xo, repo, _ = O.solve(S, cfg.rhs, _oracle_cfg(cfg, r, variant),
                          O.IterConfig(tol=1e-9, max_iters=800), method="cg")
    assert rep.converged and repo.converged
    assert rep.residual_final <= 1e-9
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8
    assert rep.precond_applications == 2 * rep.iterations


def test_kernel_class_profiling_mask(ctx):
    """set_profiling(classes=...) times only those kernel classes (the bench keeps the
    event-record overhead off the other launches); all classes when no mask is given."""
    cfg = configs.make_config("c1", 48 / 256)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    scfg = api.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    it = api.IterConfig(tol=cfg.tol, method="gmres", restart=cfg.m)
    ctx.set_profiling(True, classes=("band_solve", "lu_diag"))
    ctx.kernel_times(reset=True)
    api.solve(A, cfg.rhs, scfg, it)
    kt = ctx.kernel_times(reset=True)
    assert kt["band_solve"][1] > 0 and kt["lu_diag"][1] > 0
    assert all(n == 0 for k, (_, n) in kt.items() if k not in ("band_solve", "lu_diag"))
    ctx.set_profiling(True)
    api.solve(A, cfg.rhs, scfg, it)
    kt = ctx.kernel_times(reset=True)
    ctx.set_profiling(False)
    assert kt["krylov_vec"][1] > 0 and kt["spmv"][1] > 0 and kt["lu_diag"][1] > 0

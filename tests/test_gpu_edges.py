"""Edge cases of the hot path on the GPU (through the C-ABI) against the CPU oracle: ragged
partitions (n mod P != 0, partition sizes that are not multiples of the 128-row tile), a
single partition, a zero right-hand side, right-hand-side blocks that straddle the sweep
kernels' column groups (1 / 16 / 48), and the full-rank P = 2 known answer (SURVEY section 4:
with n_svd = k the truncated preconditioner is exact)."""
import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _cfgs(cfg, r, **kw):
    return (api.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=r, seed=cfg.seed, **kw),
            O.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=r, seed=cfg.seed, **kw))


def _solve_both(ctx, cfg, rhs, r, method, **kw):
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    gc, oc = _cfgs(cfg, r, **kw)
    m = cfg.m or 30
    x, rep, F = api.solve(A, rhs, gc, api.IterConfig(tol=cfg.tol, method=method, restart=m,
                                                     max_iters=500))
    xo, repo, Fo = O.solve(S, rhs, oc, O.IterConfig(tol=cfg.tol, restart=m, max_iters=500),
                           method=method)
    return x, rep, F, xo, repo, Fo


@pytest.mark.parametrize("name,scale,P,method", [("c1", 50 / 256, 3, "gmres"),
                                                 ("c2", 14 / 64, 5, "bicgstab"),
                                                 ("c3", 14 / 96, 3, "gmres"),
                                                 ("c1", 50 / 256, 7, "bicgstab")])
def test_ragged_partitions(ctx, name, scale, P, method):
    """n mod P != 0 (the first n mod P partitions take one more row) and no
    partition size is a multiple of 128: the last row tile of every block is partial."""
    cfg = configs.make_config(name, scale, P)
    n = cfg.matrix.n
    assert n % P != 0 and all(s % 128 != 0 for s in O.make_layout(n, P, cfg.b).sizes)
    x, rep, F, xo, repo, Fo = _solve_both(ctx, cfg, cfg.rhs, min(cfg.r, cfg.b), method)
    assert list(F.sizes) == list(O.make_layout(n, P, cfg.b).sizes)
    assert rep.converged and repo.converged and rep.residual_final <= cfg.tol
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8
    f = np.asfortranarray(np.random.default_rng(5).uniform(-1, 1, (n, 3)))
    assert _rel(F.apply_precond_T(f), O.apply_precond_T(Fo, f)) < 1e-10


def test_single_partition_is_a_direct_solve(ctx):
    """P = 1: no interfaces, no spikes; the preconditioner is A^-1 and GMRES stops after one
    step (the oracle's count)."""
    cfg = configs.make_config("c1", 40 / 256, 1)
    x, rep, F, xo, repo, Fo = _solve_both(ctx, cfg, cfg.rhs, 8, "gmres")
    assert repo.iterations == 1 and rep.iterations == repo.iterations
    assert rep.converged and rep.residual_final <= 1e-12
    assert _rel(x, xo) <= 1e-12
    m, s = rep.comm["precond-apply"]
    assert s == 0  # 4 (p - 1) n_svd n_rhs scalars per application


@pytest.mark.parametrize("method", ["gmres", "bicgstab"])
def test_zero_right_hand_side(ctx, method):
    """b = 0: x = 0 with no iterations, applications or matvecs, reported as converged."""
    cfg = configs.make_config("c1", 50 / 256, 3)
    z = np.zeros_like(cfg.rhs)
    x, rep, F, xo, repo, Fo = _solve_both(ctx, cfg, z, 8, method)
    assert repo.iterations == 0 and repo.converged and repo.precond_applications == 0
    assert rep.iterations == 0 and rep.converged
    assert rep.precond_applications == 0 and rep.matvecs == repo.matvecs
    assert not np.any(x) and not np.any(xo)


@pytest.mark.parametrize("ncols", [2, 5, 17, 49])
def test_block_solves_across_column_groups(ctx, ncols):
    """solve_block over right-hand-side blocks that straddle the sweep kernels' 16- and
    48-column groups: every column bitwise equal to its one-column solve and
    the block within 1e-12 of LAPACK's banded solve."""
    cfg = configs.make_config("c2", 16 / 64)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    F = api.factorize(ctx, A, api.SolverConfig(variant="BJ", p=cfg.P, k=cfg.b, n_svd=0))
    lay = O.make_layout(S.shape[0], cfg.P, cfg.b)
    blocks = O.extract_blocks(S, lay)
    i = 1
    R = np.asfortranarray(np.random.default_rng(ncols).uniform(-1, 1, (lay.sizes[i], ncols)))
    X = F.solve_block(i, R)
    for j in (0, ncols // 2, ncols - 1):
        assert np.array_equal(X[:, j], F.solve_block(i, R[:, j:j + 1])[:, 0]), j
    Xo = O.solve_block(O.factorize_block(blocks.A[i]), R)
    assert _rel(X, Xo) < 1e-12


@pytest.mark.parametrize("ncols", [3, 17])
def test_apply_precond_block_columns(ctx, ncols):
    """apply_precond_T on a block of right-hand sides against the oracle; the columns are
    independent: column j of the block equals the apply of column j alone to
    rounding (the one-column apply runs the FMA sweeps, the block the DMMA sweeps)."""
    cfg = configs.make_config("c2", 16 / 64)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    gc, oc = _cfgs(cfg, cfg.r)
    F = api.factorize(ctx, A, gc)
    Fo = O.factorize(S, oc)
    f = np.asfortranarray(np.random.default_rng(ncols).uniform(-1, 1, (S.shape[0], ncols)))
    X = F.apply_precond_T(f)
    assert _rel(X, O.apply_precond_T(Fo, f)) < 1e-10
    j = ncols - 1
    assert _rel(X[:, j:j + 1], F.apply_precond_T(np.asfortranarray(f[:, j:j + 1]))) < 1e-13


def test_full_rank_two_partitions_is_exact(ctx):
    """P = 2 and n_svd = k (oversample 0): the low-rank spikes are the exact spikes, so the
    truncated preconditioner inverts A and GMRES converges in one step (SURVEY section 4 KAT)."""
    cfg = configs.make_config("c1", 24 / 256, 2)
    x, rep, F, xo, repo, Fo = _solve_both(ctx, cfg, cfg.rhs, cfg.b, "gmres", oversample=0)
    assert F.n_svd == cfg.b == Fo.n_svd
    assert repo.iterations == 1 and rep.iterations == 1
    assert rep.residual_final <= 1e-10 and _rel(x, xo) <= 1e-10


def test_zero_columns_and_shape_misuse(ctx):
    """Zero-column blocks pass through as empty results; wrong shapes, dtypes and partition
    indices raise the typed errors (DimensionError / ParameterError), never a crash."""
    cfg = configs.make_config("c1", 48 / 256)
    n = cfg.matrix.n
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=8, seed=0))
    assert F.apply_precond_T(np.zeros((n, 0), order="F")).shape == (n, 0)
    assert A.spmv(np.zeros((n, 0), order="F")).shape == (n, 0)
    assert F.solve_block(0, np.zeros((F.sizes[0], 0), order="F")).shape == (F.sizes[0], 0)
    assert api.solve(A, np.zeros((n, 0), order="F"), F=F)[0].shape == (n, 0)
    with pytest.raises(api.DimensionError):
        F.apply_precond_T(np.zeros((n - 1, 1), order="F"))
    with pytest.raises(api.DimensionError):
        F.apply_precond_T(np.zeros((n, 1), dtype=np.float32, order="F"))
    with pytest.raises(api.DimensionError):
        F.apply_precond_T(np.zeros((n, 2), order="C"))
    with pytest.raises(api.ParameterError):
        F.solve_block(len(F.sizes), np.zeros((F.sizes[0], 1), order="F"))
    with pytest.raises(api.DimensionError):
        F.solve_block(0, np.zeros((F.sizes[0] + 1, 1), order="F"))
    with pytest.raises(api.ParameterError):
        api.factorize(ctx, A, api.SolverConfig(p=0, k=cfg.b, n_svd=8))
    # more right-hand sides than one batch of the multi-RHS kernels: solved in batches
    B = np.asfortranarray(np.random.default_rng(2).uniform(-1, 1, (n, 70)))
    X, rep, _ = api.solve(A, B, F=F, it=api.IterConfig(tol=1e-8, method="gmres", restart=30))
    assert rep.converged
    S = cfg.matrix.to_scipy()
    assert max(np.linalg.norm(B[:, j] - S @ X[:, j]) / np.linalg.norm(B[:, j])
               for j in range(70)) <= 1e-8 * (1 + 1e-6)

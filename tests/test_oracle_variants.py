"""The checker's LR-SPIKE-I and LR-SPIKE-OTF variants
against their SPEC examples and properties.  CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import configs


def _banded(n, k, seed, dom=1.5):
    """dense band |i - j| <= k, N(0,1) off-diagonals, diagonal dom x row sum (+1)"""
    rng = np.random.default_rng(seed)
    offs = [d for d in range(-k, k + 1) if d != 0]
    A = sp.diags([rng.standard_normal(n - abs(d)) for d in offs], offs, shape=(n, n)).tocsr()
    d = np.asarray(abs(A).sum(axis=1)).ravel() * dom + 1.0
    return (A + sp.diags(d)).tocsr()


def _tips(v, p, k):
    return O._unpack(v, p, k)


def test_matvec_lowrank_full_rank_equals_exact():
    A = _banded(120, 5, 0)
    cfg = O.SolverConfig(variant="T", p=3, k=5, n_svd=5, oversample=0, passes=4)
    F = O.factorize(A, cfg)
    lay = F.blocks.layout
    # exact tips from full spikes
    tT, tW = [], [None]
    for i in range(2):
        T = O.compute_full_spike(F.factors[i], F.blocks.B[i], O.SIDE_T)
        tT.append((T[:5], T[-5:]))
    for i in range(1, 3):
        W = O.compute_full_spike(F.factors[i], F.blocks.C[i], O.SIDE_W)
        tW.append((W[:5], W[-5:]))
    x = np.random.default_rng(1).standard_normal((2 * 5 * 3, 2))
    xt, xb = _tips(x, 3, 5)
    ye = O._pack(*O.matvec_exact(tT, tW, xt, xb))
    led = O.CommLedger()
    yl = O._pack(*O.matvec_lowrank(F, xt, xb, led))
    assert np.linalg.norm(yl - ye) / np.linalg.norm(ye) < 1e-10
    # ledger: 2 (p-1) n_svd n_rhs scalars per matvec
    assert led.stages["reduced-matvec"] == (4, 2 * 2 * 5 * 2)
    yo = O._pack(*O.matvec_otf(F, xt, xb))
    assert np.linalg.norm(yo - ye) / np.linalg.norm(ye) < 1e-11


def test_lowrank_zero_rank_is_identity_and_silent():
    A = _banded(90, 4, 2)
    F = O.factorize(A, O.SolverConfig(variant="T", p=3, k=4, n_svd=2))
    x = np.random.default_rng(3).standard_normal((24, 1))
    xt, xb = _tips(x, 3, 4)
    F2 = O.SpikeFactorization(F.blocks, F.factors, F.spT, F.spW, F.trunc, F.cfg, 0)
    for s in F2.spT + F2.spW[1:]:
        s.sigma = np.zeros_like(s.sigma)
    y = O._pack(*O.matvec_lowrank(F2, xt, xb))
    assert np.array_equal(y, x)


def test_apply_I_full_rank_is_direct_solve():
    """n_svd = k with exact tip SVDs and a tight inner tol: apply ~ A^-1 f."""
    A = _banded(150, 4, 4)
    cfg = O.SolverConfig(variant="I", p=3, k=4, n_svd=4, oversample=0, passes=4, inner_tol=1e-14)
    F = O.factorize(A, cfg)
    f = np.random.default_rng(5).standard_normal((150, 2))
    x = O.apply_precond_I(F, f)
    xd = np.linalg.solve(A.toarray(), f)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-8
    assert F.inner_solves == 1 and F.inner_iterations <= 30


def test_apply_I_block_diagonal_converges_at_half():
    A = sp.block_diag([_banded(40, 3, s) for s in range(3)]).tocsr()
    F = O.factorize(A, O.SolverConfig(variant="I", p=3, k=3, n_svd=2))
    f = np.ones((120, 1))
    x = O.apply_precond_I(F, f)
    assert np.allclose(A @ x, f, atol=1e-10)


def test_variant_ordering_I_T_BJ():
    """median outer iterations LR-SPIKE-I <= LR-SPIKE-T <= Block Jacobi."""
    its = {"I": [], "T": [], "BJ": []}
    for seed in range(10):
        A = _banded(240, 12, 100 + seed, dom=0.6)
        f = np.random.default_rng(seed).standard_normal((240, 1))
        for v in its:
            cfg = O.SolverConfig(variant=v, p=4, k=12, n_svd=3 if v != "BJ" else 0, seed=seed)
            _, rep, _ = O.solve(A, f, cfg, O.IterConfig(tol=1e-10, max_iters=500))
            its[v].append(rep.iterations)
    med = {v: float(np.median(x)) for v, x in its.items()}
    assert med["I"] <= med["T"] <= med["BJ"], med


def test_otf_solves_to_outer_tol_and_counts():
    A = _banded(300, 6, 7, dom=0.8)
    f = np.random.default_rng(8).standard_normal((300, 2))
    cfg = O.SolverConfig(variant="OTF", p=4, k=6, n_svd=3)
    x, rep, F = O.solve(A, f, cfg, O.IterConfig(tol=1e-10))
    assert rep.converged
    assert rep.residual_final <= 1e-10
    res = np.linalg.norm(A @ x - f, axis=0) / np.linalg.norm(f, axis=0)
    assert abs(res.max() - rep.residual_final) < 1e-13
    m, s = F.ledger.stages["recovery"]
    assert s % (2 * 3 * 6 * 2) == 0  # 2 (p-1) k n_rhs per recovery


def test_otf_p2_no_escalation_and_zero_coupling_shortcut():
    A = _banded(200, 5, 9)
    f = np.ones((200, 1))
    x, rep, _ = O.solve(A, f, O.SolverConfig(variant="OTF", p=2, k=5, n_svd=2),
                        O.IterConfig(tol=1e-8))
    assert rep.converged and rep.residual_final <= 1e-8
    Ab = sp.block_diag([_banded(50, 3, 1), _banded(50, 3, 2)]).tocsr()
    x, rep, _ = O.solve(Ab, np.ones((100, 1)), O.SolverConfig(variant="OTF", p=2, k=3, n_svd=2),
                        O.IterConfig(tol=1e-10))
    assert rep.iterations == 0 and rep.converged


@pytest.mark.parametrize("variant", ["I", "OTF"])
def test_variants_on_c1_structure(variant):
    cfg = configs.make_config("c1", 32 / 256)
    A = cfg.matrix.to_scipy()
    sc = O.SolverConfig(variant=variant, p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    x, rep, _ = O.solve(A, cfg.rhs, sc, O.IterConfig(tol=1e-8, restart=30), method="gmres")
    assert rep.converged and rep.residual_final <= 1e-8

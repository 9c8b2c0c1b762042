"""LR-SPIKE-I and LR-SPIKE-OTF
through the CUDA path against the oracle.

Tolerances: preconditioner applies 1e-9 relative (the LR-SPIKE-I apply contains an inner
BiCGStab to 1e-12, whose iterates differ from the oracle's by roundoff), end-to-end
solution relative difference <= 1e-8, true residual <= tol, iterations within 2.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _cfgs(cfg, variant, r=None):
    r = cfg.r if r is None else r
    return (api.SolverConfig(variant=variant, p=cfg.P, k=cfg.b, n_svd=r, seed=cfg.seed),
            O.SolverConfig(variant=variant, p=cfg.P, k=cfg.b, n_svd=r, seed=cfg.seed))


@pytest.mark.parametrize("name,scale,r", [("c1", 48 / 256, 8), ("c2", 16 / 64, 16)])
def test_apply_precond_I_matches_oracle(ctx, name, scale, r):
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    gc, oc = _cfgs(cfg, "I", r)
    F = api.factorize(ctx, A, gc)
    Fo = O.factorize(S, oc)
    f = np.asfortranarray(np.random.default_rng(2).uniform(-1, 1, (S.shape[0], 3)))
    assert _rel(F.apply_precond_I(f), O.apply_precond_I(Fo, f)) < 1e-9
    # the T apply of the same factorization is still available
    assert _rel(F.apply_precond_T(f), O.apply_precond_T(Fo, f)) < 1e-10


@pytest.mark.parametrize("name,scale,method", [("c1", 48 / 256, "gmres"),
                                               ("c2", 16 / 64, "bicgstab")])
@pytest.mark.parametrize("variant", ["I", "OTF"])
def test_variant_solve_parity(ctx, name, scale, method, variant):
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    gc, oc = _cfgs(cfg, variant)
    it = api.IterConfig(tol=cfg.tol, method=method, restart=cfg.m or 30, max_iters=500)
    x, rep, F = api.solve(A, cfg.rhs, gc, it)
    xo, repo, Fo = O.solve(S, cfg.rhs, oc, O.IterConfig(tol=cfg.tol, restart=cfg.m or 30,
                                                        max_iters=500), method=method)
    assert rep.converged and repo.converged
    assert rep.residual_final <= cfg.tol
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8
    if variant == "I":
        assert rep.inner_solves == rep.precond_applications
        assert rep.inner_iterations > 0
        assert abs(rep.inner_iterations - repo.inner_iterations) <= 2 + 0.05 * repo.inner_iterations
        # ledger: T-style messages + 2 (p-1) r n_rhs per inner matvec
        m, s = rep.comm["recovery"]
        assert s == 2 * (cfg.P - 1) * F.n_svd * rep.precond_applications
    else:
        m, s = rep.comm["reduced-matvec"]
        assert s > 0 and s % (2 * (cfg.P - 1) * cfg.b) == 0  # 2 (p-1) k n_rhs per matvec


def test_otf_zero_coupling_shortcut(ctx):
    blocks = [sp.diags([-1.0, 4.0, -1.0], [-1, 0, 1], shape=(60, 60)) for _ in range(3)]
    Z = sp.block_diag(blocks).tocsr()
    A = api.CsrMatrix(ctx, Z.shape[0], Z.indptr, Z.indices, Z.data)
    b = np.ones((Z.shape[0], 1))
    x, rep, _ = api.solve(A, b, api.SolverConfig(variant="OTF", p=3, k=2, n_svd=1),
                          api.IterConfig(tol=1e-12))
    assert rep.converged and rep.iterations == 0
    assert _rel(Z @ x, b) < 1e-13


@pytest.mark.parametrize("variant", ["I", "OTF"])
def test_complex_variants(ctx, variant):
    cfg = configs.make_config("c5", 16 / 80, P=4)
    Az = cfg.system(2)
    S = Az.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, Az)
    b = np.asfortranarray(cfg.rhs[:, :2].astype(np.complex128))
    gc, oc = _cfgs(cfg, variant, 16)
    it = api.IterConfig(tol=1e-9, method="gmres", restart=40, max_iters=800)
    x, rep, F = api.solve(A, b, gc, it)
    xo, repo, _ = O.solve(S, b, oc, O.IterConfig(tol=1e-9, restart=40, max_iters=800),
                          method="gmres")
    assert rep.converged and repo.converged
    assert abs(rep.iterations - repo.iterations) <= 2
    assert _rel(x, xo) <= 1e-8


def test_reduced_system_operators_match_oracle(ctx):
    """matvec_lowrank / matvec_exact / apply_truncated_precond on
    ReducedVector blocks; the preconditioner inverts the assembled truncated system."""
    cfg = configs.make_config("c1", 48 / 256)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    gc, oc = _cfgs(cfg, "T", 8)
    F = api.factorize(ctx, A, gc)
    Fo = O.factorize(S, oc)
    p, k = cfg.P, cfg.b
    xr = np.asfortranarray(np.random.default_rng(6).standard_normal((2 * k * p, 3)))
    xt, xb = O._unpack(xr, p, k)
    assert _rel(F.matvec_lowrank(xr), O._pack(*O.matvec_lowrank(Fo, xt, xb))) < 1e-12
    assert _rel(F.matvec_exact(xr), O._pack(*O.matvec_otf(Fo, xt, xb))) < 1e-12
    g = F.apply_truncated_precond(xr)
    assert _rel(g, O._pack(*O.apply_truncated_precond(Fo.trunc, xt, xb))) < 1e-11


def test_cli_solve_with_reorder_pipeline(tmp_path):
    """Matrix Market in, reorder pipeline, GPU solve, solution mapped back."""
    import json

    from paper_2504_11167_b200 import cli, reorder
    from paper_2504_11167_b200.configs import Csr

    S = configs.make_config("c1", 48 / 256).matrix.to_scipy()
    n = S.shape[0]
    p = np.random.default_rng(2).permutation(n)
    Sp = sp.csr_matrix((S.data, S.indices, S.indptr), shape=S.shape)[p][:, p].tocsr()
    Sp.sort_indices()
    src = tmp_path / "a.mtx"
    reorder.write_matrix_market(str(src), Csr(n, Sp.indptr.astype(np.int64),
                                              Sp.indices.astype(np.int64), Sp.data))
    rep_path, x_path = tmp_path / "r.json", tmp_path / "x.npy"
    assert cli.main(["solve", "--in", str(src), "--rhs", "ones", "--variant", "t", "-p", "4",
                     "--nsvd", "8", "--tol", "1e-9", "--method", "gmres", "--reorder",
                     "--report", str(rep_path), "--x-out", str(x_path)]) == 0
    r = json.load(open(rep_path))
    assert r["converged"] and r["residual_final"] <= 1e-8
    x = np.load(x_path)
    assert _rel(Sp @ x, np.ones((n, 1))) <= 1e-8

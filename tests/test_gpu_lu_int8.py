"""The INT8-sliced (Ozaki) two-step LU update on the tcgen05 tensor cores (csrc/lu_i8.cu)
against the FP64 DMMA update and the oracle.  Tolerances: factor tiles within 1e-12 of
the DMMA factors (relative to the partition's largest tile entry -- the same bar as the
DMMA-vs-LAPACK kernel parity), solves at the north_star bars."""
import os

import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs
from paper_2504_11167_b200.configs import Csr

pytestmark = pytest.mark.gpu


def _factor(ctx, csr, cfg, i8, quad=False):
    old = {k: os.environ.get(k) for k in ("LRS_LU_I8", "LRS_LU_QUAD")}
    os.environ["LRS_LU_I8"] = "1" if i8 else "0"
    os.environ["LRS_LU_QUAD"] = "1" if quad else "0"
    try:
        A = api.CsrMatrix.from_csr(ctx, csr)
        return api.factorize(ctx, A, api.SolverConfig(variant="BJ", p=cfg.P, k=cfg.b, n_svd=0))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v


def _compare(ctx, csr, cfg, quad=False):
    F8 = _factor(ctx, csr, cfg, True, quad)
    F64 = _factor(ctx, csr, cfg, False)
    assert F8.info["lu_int8"] == 1 and F64.info["lu_int8"] == 0
    if not F8.info["pivoted"]:
        assert F8.info["lu_pairs"] == (4 if quad else 2)
    worst = 0.0
    for i in range(cfg.P):
        a, b = F8.tiles(i), F64.tiles(i)
        worst = max(worst, float(np.max(np.abs(a - b)) / np.max(np.abs(b))))
    return worst


def test_i8_peak_positive(ctx):
    tops = ctx.i8_peak_tops()
    assert 500.0 < tops < 20000.0


@pytest.mark.parametrize("name,scale", [("c2", 0.5), ("c3", 24 / 96), ("c4", 0.05)])
def test_int8_update_matches_dmma(ctx, name, scale):
    cfg = configs.make_config(name, scale)
    assert -(-cfg.b // 128) >= 3  # the pair schedule (and so the INT8 update) is in play
    assert _compare(ctx, cfg.system(0), cfg) <= 1e-12


@pytest.mark.parametrize("name,scale", [("c2", 0.5), ("c4", 0.05)])
def test_int8_quad_update_matches_dmma(ctx, name, scale):
    """LRS_LU_QUAD=1: four steps (K = 512) per INT8 update, DMMA look-ahead inside the quad."""
    cfg = configs.make_config(name, scale)
    assert -(-cfg.b // 128) >= 8
    assert _compare(ctx, cfg.system(0), cfg, quad=True) <= 1e-12


@pytest.mark.parametrize("e", [-300, 300])
def test_int8_update_far_exponents(ctx, e):
    """Uniformly scaled matrices: the per-row / per-column exponents carry the scale."""
    cfg = configs.make_config("c2", 0.5)
    m = cfg.matrix
    scaled = Csr(m.n, m.row_ptr, m.col_idx, m.values * 2.0 ** e)
    assert _compare(ctx, scaled, cfg) <= 1e-12


def test_int8_graded_rows(ctx):
    """Rows graded over 2^+-20 (a slowly varying diagonal scaling keeps dominance)."""
    cfg = configs.make_config("c2", 0.5)
    S = cfg.matrix.to_scipy().tocsr()
    n = S.shape[0]
    d = 2.0 ** np.round(20 * np.sin(np.arange(n) / 3000.0))
    import scipy.sparse as sp
    G = (sp.diags(d) @ S @ sp.diags(1.0 / d)).tocsr()
    G.sort_indices()
    csr = Csr(n, G.indptr.astype(np.int64), G.indices.astype(np.int64), G.data)
    assert _compare(ctx, csr, cfg) <= 1e-12


def test_int8_solve_parity_with_oracle(ctx):
    cfg = configs.make_config("c2", 0.5)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    scfg = api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=500)
    F = api.factorize(ctx, A, scfg)
    assert F.info["lu_int8"] == 1
    x, rep, _ = api.solve(A, np.asfortranarray(cfg.rhs), it=it, F=F)
    ocfg = O.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    xo, ro, _ = O.solve(S, cfg.rhs, ocfg, O.IterConfig(tol=cfg.tol, restart=cfg.m or 30,
                                                       max_iters=500), method=cfg.method)
    assert rep.converged and rep.residual_final <= cfg.tol
    assert abs(rep.iterations - ro.iterations) <= 2
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-8

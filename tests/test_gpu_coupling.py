"""spike_mode = coupling on the GPU against the oracle's coupling_spike_svd (north_star
setup (1): truncated rank-r SVD of the coupling blocks B_i / C_i, then the low-rank spikes
by multi-RHS padded solves against the singular vectors).

Bars: the spike operators u S v to 1e-9 and sigma to 1e-10 (basis independent: the range
finder fixes the subspace, the SVD basis inside it may differ), the preconditioner apply
to 1e-10, solves at the north_star bars (iterations within 2, x within 1e-8, residual <= tol).
The iteration counts against the default spike mode are printed (SURVEY.md D4 measured
37 vs 16-21 on the c1 structure)."""
import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _cfgs(cfg, mode):
    return (api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed, spike_mode=mode),
            O.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed, spike_mode=mode))


@pytest.mark.parametrize("name,scale,shift", [("c1", 48 / 256, None), ("c2", 16 / 64, None),
                                              ("c5", 16 / 80, 2)])
def test_coupling_spikes_and_apply_match_oracle(ctx, name, scale, shift):
    cfg = configs.make_config(name, scale, P=4 if name == "c5" else None)
    csr = cfg.system(shift) if shift is not None else cfg.matrix
    S = csr.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, csr)
    g, o = _cfgs(cfg, "coupling")
    F = api.factorize(ctx, A, g)
    Fo = O.factorize(S, o)
    assert F.n_svd == Fo.n_svd
    for i, side in ((0, api.SIDE_T), (1, api.SIDE_W), (cfg.P - 2, api.SIDE_T)):
        u, s, v = F.spike(i, side)
        so = Fo.spT[i] if side == api.SIDE_T else Fo.spW[i]
        assert _rel(s, so.sigma) < 1e-10
        assert _rel((u * s) @ v, (so.u * so.sigma) @ so.v) < 1e-9
    rng = np.random.default_rng(4)
    f = rng.uniform(-1, 1, (S.shape[0], 2))
    if np.iscomplexobj(S.data):
        f = f + 1j * rng.uniform(-1, 1, f.shape)
    f = np.asfortranarray(f)
    assert _rel(F.apply_precond_T(f), O.apply_precond_T(Fo, f)) < 1e-10


@pytest.mark.parametrize("name,scale,method", [("c1", 48 / 256, "gmres"),
                                               ("c1", 96 / 256, "gmres"),
                                               ("c2", 16 / 64, "bicgstab"),
                                               ("c2", 24 / 64, "bicgstab")])
def test_coupling_solve_parity(ctx, name, scale, method):
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    it = api.IterConfig(tol=cfg.tol, method=method, restart=cfg.m or 30, max_iters=500)
    ito = O.IterConfig(tol=cfg.tol, restart=cfg.m or 30, max_iters=500)
    its = {}
    for mode in ("spike", "coupling"):
        g, o = _cfgs(cfg, mode)
        x, rep, _ = api.solve(A, cfg.rhs, g, it)
        xo, repo, _ = O.solve(S, cfg.rhs, o, ito, method=method)
        assert rep.converged and rep.residual_final <= cfg.tol
        assert abs(rep.iterations - repo.iterations) <= 2
        assert _rel(x, xo) <= 1e-8
        its[mode] = (rep.iterations, repo.iterations)
    print(f"{name}@{scale:.3f} {method}: iterations (gpu, oracle) spike {its['spike']}, "
          f"coupling {its['coupling']}")
    assert its["spike"][0] <= its["coupling"][0]


def test_coupling_mode_rejects_unknown(ctx):
    cfg = configs.make_config("c1", 48 / 256)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    with pytest.raises(api.ParameterError):
        api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, spike_mode="x"))

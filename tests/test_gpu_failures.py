"""Failure branches on the GPU, on the constructed inputs of
tests/failure_cases.py, against the oracle:

* the r-halving retry: n_svd = 2 gives a singular interface matrix K, factorize halves it
  once and succeeds at n_svd = 1 (the solve then matches the oracle's);
* IllConditionedInterfaceError after the retry, with its payload (interface index,
  cond_1 > 1e12) through the C-ABI's lrs_last_error -- and from build_truncated_precond on
  explicit spikes whose K is exactly singular;
* rank collapse: couplings of rank 3 < n_svd = 8, sigma_4..8 truncated to 0, the flag set
  in the factorization info, the solve still matches the oracle;
* BiCGStab breakdown (omega = 0 on a skew-symmetric operator) through lrs_krylov: the
  BreakdownError carries the partial x and the report.
"""
import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api
from tests import failure_cases as FC

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("seed", [3, 5, 11])
def test_r_halving_retry_on_gpu(ctx, seed):
    A, k = FC.ill_conditioned_interface(True)
    Ad = api.CsrMatrix.from_csr(ctx, A)
    F = api.factorize(ctx, Ad, api.SolverConfig(p=2, k=k, n_svd=2, seed=seed))
    assert F.n_svd == 1 and F.info["max_interface_cond"] < 1e12
    Fo = O.factorize(A.to_scipy(), O.SolverConfig(p=2, k=k, n_svd=2, seed=seed))
    assert Fo.n_svd == 1
    b = np.asfortranarray(np.random.default_rng(seed).uniform(-1, 1, (A.n, 1)))
    x, rep, _ = api.solve(Ad, b, it=api.IterConfig(tol=1e-10, method="bicgstab"), F=F)
    xo, repo, _ = O.solve(A.to_scipy(), b, O.SolverConfig(p=2, k=k, n_svd=2, seed=seed),
                          O.IterConfig(tol=1e-10), method="bicgstab", F=Fo)
    assert rep.converged and rep.residual_final <= 1e-10
    assert abs(rep.iterations - repo.iterations) <= 2 and _rel(x, xo) <= 1e-8


@pytest.mark.parametrize("seed", [3, 5, 11])
def test_ill_conditioned_interface_error_payload(ctx, seed):
    A, k = FC.ill_conditioned_interface(False)
    Ad = api.CsrMatrix.from_csr(ctx, A)
    with pytest.raises(api.IllConditionedInterfaceError) as e:
        api.factorize(ctx, Ad, api.SolverConfig(p=2, k=k, n_svd=4, seed=seed))
    assert e.value.interface_index == 0 and e.value.cond_estimate > 1e12


def test_build_truncated_precond_singular_interface(ctx):
    """K = v_W u_{T,b} exactly singular: u tips on axes {0,1}, v_W rows on axes {1,2}."""
    k, r, n_i = 4, 2, 10
    uT = np.zeros((n_i, r))
    uT[n_i - k + 0, 0] = uT[n_i - k + 1, 1] = 1.0
    uW = np.zeros((n_i, r))
    uW[2, 0] = uW[3, 1] = 1.0
    vT = np.eye(r, k)
    vW = np.zeros((r, k))
    vW[0, 1] = vW[1, 2] = 1.0
    s = np.array([1.0, 0.5])
    with pytest.raises(api.IllConditionedInterfaceError) as e:
        api.build_truncated_precond(ctx, [(uT, s, vT)], [(uW, s, vW)], k)
    assert e.value.interface_index == 0 and e.value.cond_estimate > 1e12
    # the same spikes with an invertible K are accepted and match the oracle's Woodbury
    vW = np.zeros((r, k))
    vW[0, 0] = vW[1, 1] = 1.0
    P = api.build_truncated_precond(ctx, [(uT, s, vT)], [(uW, s, vW)], k)
    spT = [O.LowRankSpike(uT, s, vT, O.SIDE_T)]
    spW = [None, O.LowRankSpike(uW, s, vW, O.SIDE_W)]
    Po = O.build_truncated_precond(spT, spW, k)
    g = np.random.default_rng(2).uniform(-1, 1, (2 * k * 2, 3))
    top, bot = [g[0:k], g[2 * k:3 * k]], [g[k:2 * k], g[3 * k:4 * k]]
    xt, xb = O.apply_truncated_precond(Po, top, bot)
    ref = np.concatenate([xt[0], xb[0], xt[1], xb[1]])
    assert _rel(P.apply(g), ref) <= 1e-13


def test_rank_collapse_on_gpu(ctx):
    A, g = FC.rank_deficient_coupling()
    Ad = api.CsrMatrix.from_csr(ctx, A)
    cfg = api.SolverConfig(p=4, k=g, n_svd=8, seed=0)
    F = api.factorize(ctx, Ad, cfg)
    assert F.info["rank_collapsed"] == 1 and F.n_svd == 8
    _, s, _ = F.spike(0, api.SIDE_T)
    assert np.count_nonzero(s) == 3
    b = np.asfortranarray(np.random.default_rng(0).uniform(-1, 1, (A.n, 1)))
    x, rep, _ = api.solve(Ad, b, it=api.IterConfig(tol=1e-8, method="gmres", restart=30), F=F)
    xo, repo, Fo = O.solve(A.to_scipy(), b, O.SolverConfig(p=4, k=g, n_svd=8, seed=0),
                           O.IterConfig(tol=1e-8, restart=30), method="gmres")
    assert Fo.rank_collapsed
    assert rep.converged and rep.residual_final <= 1e-8
    assert abs(rep.iterations - repo.iterations) <= 2 and _rel(x, xo) <= 1e-8


def test_bicgstab_breakdown_partial_result_through_c_abi(ctx):
    import torch

    n = 64  # block-diagonal skew-symmetric [[0, -1], [1, 0]] blocks: (t, s) = 0 -> omega = 0

    def skew(x, y):
        y[0::2] = -x[1::2]
        y[1::2] = x[0::2]

    b = np.zeros((n, 1), order="F")
    b[0::2] = 1.0
    with pytest.raises(api.BreakdownError) as e:
        api.krylov(ctx, skew, b, api.IterConfig(tol=1e-14, max_iters=10, method="bicgstab"))
    assert e.value.report.breakdown and e.value.x is not None
    assert np.all(np.isfinite(np.asarray(e.value.x)))
    # the oracle raises at the same point with the same partial iterate
    A = np.zeros((n, n))
    for i in range(0, n, 2):
        A[i, i + 1], A[i + 1, i] = -1.0, 1.0
    with pytest.raises(O.BreakdownError) as eo:
        O.bicgstab(lambda v: A @ v, lambda v: v, b,
                   O.IterConfig(tol=1e-14, max_iters=10, breakdown_eps=1e-30))
    assert _rel(np.asarray(e.value.x), eo.value.x) <= 1e-14
    del torch

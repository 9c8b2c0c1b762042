"""Failure semantics of the oracle on constructed inputs (tests/failure_cases.py): the
r-halving retry, IllConditionedInterfaceError with its payload,
rank collapse.  The GPU runs the same inputs in test_gpu_failures.py."""
import numpy as np
import pytest

from oracle import lrspike_oracle as O
from tests import failure_cases as FC


@pytest.mark.parametrize("seed", [3, 5, 11])
def test_r_halving_retry_succeeds(seed):
    A, k = FC.ill_conditioned_interface(True)
    S = A.to_scipy()
    with pytest.raises(O.IllConditionedInterfaceError):  # at n_svd = 2 directly
        O.build_truncated_precond(*O._build_spikes(O.extract_blocks(S, O.make_layout(A.n, 2, k)),
                                                   [O.factorize_block(b) for b in
                                                    O.extract_blocks(S, O.make_layout(A.n, 2, k)).A],
                                                   O.SolverConfig(p=2, k=k, n_svd=2, seed=seed),
                                                   2, k)[:2], k)
    F = O.factorize(S, O.SolverConfig(p=2, k=k, n_svd=2, seed=seed))
    assert F.n_svd == 1
    b = np.random.default_rng(seed).uniform(-1, 1, (A.n, 1))
    x, rep, _ = O.solve(S, b, O.SolverConfig(p=2, k=k, n_svd=2, seed=seed),
                        O.IterConfig(tol=1e-10), method="bicgstab", F=F)
    assert rep.converged and rep.residual_final <= 1e-10


@pytest.mark.parametrize("seed", [3, 5, 11])
def test_ill_conditioned_interface_raises_after_halving(seed):
    A, k = FC.ill_conditioned_interface(False)
    with pytest.raises(O.IllConditionedInterfaceError) as e:
        O.factorize(A.to_scipy(), O.SolverConfig(p=2, k=k, n_svd=4, seed=seed))
    assert e.value.interface_index == 0 and e.value.cond_estimate > O.COND_LIMIT


def test_rank_collapse_flag_and_convergence():
    A, g = FC.rank_deficient_coupling()
    S = A.to_scipy()
    cfg = O.SolverConfig(p=4, k=g, n_svd=8, seed=0)
    F = O.factorize(S, cfg)
    assert F.rank_collapsed and F.n_svd == 8
    for sp_ in F.spT + F.spW[1:]:
        assert np.count_nonzero(sp_.sigma) == 3 and sp_.rank_collapsed
    b = np.random.default_rng(0).uniform(-1, 1, (A.n, 1))
    x, rep, _ = O.solve(S, b, cfg, O.IterConfig(tol=1e-8, restart=30), method="gmres", F=F)
    assert rep.converged and rep.residual_final <= 1e-8

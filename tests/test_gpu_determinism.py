"""Race detection by repetition (compute-sanitizer is closed on the GPU pool: its runs left
GPUs needing a reset; profiles/r02_sanitizer.txt).  Every kernel of the path is
deterministic by construction -- fixed-order reductions, one writer per element, the
ticket-ordered dataflow sweeps, the INT8 update's single L2 reduction per element -- so a
race (a missed hand-off in the mailbox / epoch-flag protocol, a 2-CTA cluster panel
writing before its partner read, a TMEM slot reused early) shows up as a bitwise
difference between repeated runs on identical inputs:

* the band factor tiles of repeated factorizations (INT8 tcgen05 update with its TMEM slot
  ring and TMA ring, cluster panels, look-ahead streams) on the c2 structure (b = 576);
* repeated preconditioner applies (one-RHS mailbox sweeps + interface + recovery), 100x;
* the 48-column spike sweeps (adjoint DMMA kernels), through the spikes of each factorization;
* repeated solves (SpMV, multi-dot, GMRES / BiCGStab vector kernels).
"""
import numpy as np
import pytest

from paper_2504_11167_b200 import api, configs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,scale", [("c2", 24 / 64), ("c3", 24 / 96), ("c1", 96 / 256)])
def test_repeated_factorizations_bitwise(ctx, name, scale):
    cfg = configs.make_config(name, scale)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    scfg = api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    ref = api.factorize(ctx, A, scfg)
    t0 = [ref.tiles(i) for i in (0, cfg.P - 1)]
    s0 = ref.spike(0, api.SIDE_T)
    for _ in range(4):
        F = api.factorize(ctx, A, scfg)
        for i, t in zip((0, cfg.P - 1), t0):
            assert np.array_equal(F.tiles(i), t)
        s = F.spike(0, api.SIDE_T)
        assert all(np.array_equal(a, b) for a, b in zip(s, s0))
        del F


@pytest.mark.parametrize("name,scale", [("c2", 24 / 64), ("c1", 96 / 256)])
def test_repeated_applies_and_solves_bitwise(ctx, name, scale):
    import torch

    cfg = configs.make_config(name, scale)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
    f = np.asfortranarray(configs.vector("uniform", 5, cfg.matrix.n))
    fd = torch.from_numpy(f.T.copy()).cuda().t()
    torch.cuda.synchronize()
    # the library runs on its own stream: wait for it before torch reads the output
    y0 = F.apply_precond_T(fd)
    ctx.synchronize()
    y0 = y0.clone()
    torch.cuda.synchronize()
    for _ in range(100):
        y = F.apply_precond_T(fd)
        ctx.synchronize()
        assert torch.equal(y, y0)
    it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=500)
    x0, r0, _ = api.solve(A, cfg.rhs, it=it, F=F)
    for _ in range(3):
        x, r, _ = api.solve(A, cfg.rhs, it=it, F=F)
        assert np.array_equal(x, x0) and r.residual_history == r0.residual_history

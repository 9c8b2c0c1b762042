"""Partial-pivoting path timing on the c2 structure with rows scaled by 10^U[-1.5, 1.5]
(dgbtrf interchanges in every block) -- development aid."""
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
cfg = configs.make_config("c2", scale)
S = cfg.matrix.to_scipy()
rng = np.random.default_rng(0)
S = (sp.diags(10.0 ** rng.uniform(-1.5, 1.5, S.shape[0])) @ S).tocsr()
S.sort_indices()
ctx = api.Context(0)
A = api.CsrMatrix(ctx, S.shape[0], S.indptr, S.indices, S.data)
for variant, r in (("BJ", 0), ("T", cfg.r)):
    F = api.factorize(ctx, A, api.SolverConfig(variant=variant, p=cfg.P, k=cfg.b, n_svd=r,
                                               seed=cfg.seed))
    inf = F.info
    f = np.asfortranarray(cfg.rhs)
    F.apply(f)
    ctx.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        F.apply(f)
    ctx.synchronize()
    ta = (time.perf_counter() - t) / 5
    it = api.IterConfig(tol=1e-8, method="gmres", restart=30, max_iters=500)
    x, rep, _ = api.solve(A, f, it=it, F=F)
    print(variant, {"pivoted": inf["pivoted"], "t_lu": inf["t_lu"], "t_spikes": inf["t_spikes"],
                    "wu": inf["wu"], "factor_GB": inf["factor_bytes"] / 1e9,
                    "apply_ms": ta * 1e3, "iters": rep.iterations, "conv": rep.converged,
                    "t_solve": rep.wall_time}, flush=True)

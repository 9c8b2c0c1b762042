"""API misuse probes: zero columns, wrong shapes, wrong dtypes -- each must raise a typed
lrspike error or return an empty result; none may crash the process."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

cfg = configs.make_config("c1", 48 / 256)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=8, seed=0))
n = cfg.matrix.n


def probe(tag, fn):
    try:
        r = fn()
        print(tag, "->", type(r).__name__, getattr(r, "shape", None), flush=True)
    except api.Error as e:
        print(tag, "-> raised", type(e).__name__, str(e)[:80], flush=True)
    except Exception as e:  # noqa: BLE001
        print(tag, "-> raised (untyped)", type(e).__name__, str(e)[:80], flush=True)


probe("apply 0 cols", lambda: F.apply_precond_T(np.zeros((n, 0), order="F")))
probe("apply wrong rows", lambda: F.apply_precond_T(np.zeros((n - 1, 1), order="F")))
probe("apply float32", lambda: F.apply_precond_T(np.zeros((n, 1), dtype=np.float32, order="F")))
probe("apply C order 2 cols", lambda: F.apply_precond_T(np.zeros((n, 2), order="C")))
probe("spmv 0 cols", lambda: A.spmv(np.zeros((n, 0), order="F")))
probe("solve_block 0 cols", lambda: F.solve_block(0, np.zeros((F.sizes[0], 0), order="F")))
probe("solve_block bad partition", lambda: F.solve_block(99, np.zeros((F.sizes[0], 1), order="F")))
probe("solve_block wrong rows", lambda: F.solve_block(0, np.zeros((F.sizes[0] + 1, 1), order="F")))
probe("solve 0 cols", lambda: api.solve(A, np.zeros((n, 0), order="F"), F=F)[0])
probe("solve 70 cols", lambda: api.solve(A, np.ones((n, 70), order="F"), F=F,
                                         it=api.IterConfig(tol=1e-8, method="gmres", restart=30))[1].iterations)
probe("factorize p > n/k", lambda: api.factorize(ctx, A, api.SolverConfig(p=4000, k=cfg.b, n_svd=8)))
probe("factorize n_svd > k", lambda: api.factorize(ctx, A, api.SolverConfig(p=4, k=cfg.b, n_svd=cfg.b + 1)))
probe("factorize p = 0", lambda: api.factorize(ctx, A, api.SolverConfig(p=0, k=cfg.b, n_svd=8)))
probe("factorize k = 0 on a banded matrix", lambda: api.factorize(ctx, A, api.SolverConfig(p=4, k=0, n_svd=0, variant="BJ")))
probe("empty matrix", lambda: api.CsrMatrix(ctx, 0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0)))
print("alive", flush=True)

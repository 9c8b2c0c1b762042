"""One small LR-SPIKE factorize + solve for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): c1 structure (FMA dataflow sweeps, DMMA band LU) or c2 structure at
24^3 (b = 576: the INT8 tcgen05 two-step update, 2-CTA cluster panels, mailbox sweeps,
48-column spike sweeps), plus one complex128 c5 solve."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
ctx = api.Context(0)
if name == "c5":
    cfg = configs.make_config("c5", 12 / 80, P=4)
    csr = cfg.system(1)
    rhs = np.asfortranarray(cfg.rhs[:, :2].astype(np.complex128))
else:
    cfg = configs.make_config(name, {"c1": 48 / 256, "c2": 24 / 64}[name])
    csr, rhs = cfg.matrix, cfg.rhs
A = api.CsrMatrix.from_csr(ctx, csr)
it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=40)
x, rep, F = api.solve(A, rhs, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed), it)
print(f"{name}: iterations {rep.iterations} residual {rep.residual_final:.2e} "
      f"lu_int8 {F.info['lu_int8']} launches {ctx.launches}")

"""Per-class kernel time of a few GMRES(40) iterations of config c5 (one shift, 16 RHS)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

cfg = configs.make_config("c5", float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.system(0))
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
b = np.asfortranarray(cfg.rhs.astype(np.complex128))
it = api.IterConfig(tol=cfg.tol, method="gmres", restart=cfg.m, max_iters=80)
ctx.set_profiling(True)
ctx.kernel_times(reset=True)
x, rep, _ = api.solve(A, b, it=it, F=F)
ctx.synchronize()
kt = ctx.kernel_times(reset=True)
print("iterations", rep.iterations, "wall", rep.wall_time)
for k, (ms, n) in kt.items():
    if n:
        print(f"{k:20s} {ms:10.2f} ms {n:6d} launches")

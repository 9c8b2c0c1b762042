"""Diagnose solve-phase host gaps: time 71 applies vs a full BiCGStab solve (c2)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2504_11167_b200 import api, configs  # noqa: E402

ctx = api.Context(0)
cfg = configs.make_config("c2", float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
f = torch.from_numpy(np.asfortranarray(cfg.rhs)).cuda()
x = torch.empty_like(f)
torch.cuda.synchronize()
for _ in range(3):
    F.apply_precond_T(f, x)
ctx.synchronize()
t = time.perf_counter()
for _ in range(71):
    F.apply_precond_T(f, x)
ctx.synchronize()
print("71 applies", time.perf_counter() - t)
it = api.IterConfig(tol=cfg.tol, method="bicgstab")
for rep in range(3):
    t = time.perf_counter()
    xs, r, _ = api.solve(A, f, it=it, F=F, x_out=x)
    ctx.synchronize()
    print("solve", time.perf_counter() - t, r.wall_time, r.iterations)

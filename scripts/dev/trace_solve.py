import os, sys
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_2504_11167_b200 import api, configs
cfg = configs.make_config("c2")
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ctx = api.Context(0, st.cuda_stream)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
bd = torch.from_numpy(np.asfortranarray(cfg.rhs)).cuda(); xd = torch.empty_like(bd)
it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=2000)
for k in range(6):
    print("=== solve", k, file=sys.stderr, flush=True)
    x, r, _ = api.solve(A, bd, it=it, F=F, x_out=xd)
    print("solve", "%.1f ms" % (1e3 * r.wall_time), file=sys.stderr, flush=True)

import os, sys, time, re
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2504_11167_b200 import api, configs
ctx = api.Context(0)
cfg = configs.make_config("c2", 1.0)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
f = torch.from_numpy(np.asfortranarray(cfg.rhs)).cuda(); x = torch.empty_like(f)
torch.cuda.synchronize()
it = api.IterConfig(tol=cfg.tol, method="bicgstab")
for rep in range(8):
    t = time.perf_counter()
    F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
    t1 = time.perf_counter()
    xs, r, _ = api.solve(A, f, it=it, F=F, x_out=x)
    ctx.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep} fact {t1-t:.3f} (lu {F.info['t_lu']:.3f} spk {F.info['t_spikes']:.3f}) solve {t2-t1:.3f} ({r.wall_time:.3f})", flush=True)
    del F

"""FP64 vs FP32-factor apply on c2 (development aid)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2504_11167_b200 import api, configs  # noqa: E402

cfg = configs.make_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = api.Context(0, st.cuda_stream)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
bd = torch.from_numpy(np.asfortranarray(cfg.rhs)).cuda()
xd = torch.empty_like(bd)
for fp32 in (False, True, False, True):
    F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed,
                                               factor_fp32=fp32))
    F.apply_precond_T(bd, xd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        F.apply_precond_T(bd, xd)
    e1.record(st)
    torch.cuda.synchronize()
    ta = e0.elapsed_time(e1) / 20
    it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=2000)
    x, rep, _ = api.solve(A, bd, it=it, F=F, x_out=xd)
    print({"fp32": fp32, "apply_ms": ta, "apply_GBps": F.info["apply_bytes"] / ta / 1e6,
           "iters": rep.iterations, "t_solve": rep.wall_time, "t_fact": F.info["t_factorize"],
           "res": rep.residual_final}, flush=True)
    del F

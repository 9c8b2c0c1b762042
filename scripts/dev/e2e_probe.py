"""Breakdown of the e2e (host-buffer) step of bench.py (development aid)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2504_11167_b200 import api, configs  # noqa: E402

cfg = configs.make_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
ctx = api.Context(0, torch.cuda.current_stream().cuda_stream)
csr = cfg.matrix
scfg = api.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=2000)
b = np.asfortranarray(cfg.rhs)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A2 = api.CsrMatrix(ctx, csr.n, csr.row_ptr, csr.col_idx, csr.values)
    ctx.synchronize()
    t1 = time.perf_counter()
    F2 = api.factorize(ctx, A2, scfg)
    ctx.synchronize()
    t2 = time.perf_counter()
    xh, r, _ = api.solve(A2, b, it=it, F=F2)
    t3 = time.perf_counter()
    del F2
    t4 = time.perf_counter()
    del A2
    t5 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms factorize {1e3*(t2-t1):.1f} (gpu {1e3*F2_info if False else 0}) "
          f"solve {1e3*(t3-t2):.1f} (gpu {1e3*r.wall_time:.1f}) free_fact {1e3*(t4-t3):.1f} "
          f"free_mat {1e3*(t5-t4):.1f} total {1e3*(t5-t0):.1f}", flush=True)
# profiling overhead
for prof in (False, True, False, True):
    ctx.set_profiling(prof)
    bd = torch.from_numpy(b).cuda()
    xd = torch.empty_like(bd)
    A = api.CsrMatrix.from_csr(ctx, csr)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    F = api.factorize(ctx, A, scfg)
    x, r, _ = api.solve(A, bd, it=it, F=F, x_out=xd)
    torch.cuda.synchronize()
    print("profiling", prof, f"{1e3*(time.perf_counter()-t0):.1f} ms", F.info["t_lu"], r.wall_time,
          flush=True)
    del F

"""Wall-clock split of bench.py's e2e step on c3 P=64 (page-locked host buffers): upload, factorize
(wall vs the library's CUDA events), solve (wall vs events), frees."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

cfg = configs.make_config("c3", 1.0, 64)
ctx = api.Context(0)
csr = cfg.matrix


def pinned(a):
    t = torch.empty(a.size, dtype=torch.from_numpy(a[:0].copy()).dtype, pin_memory=True)
    v = t.numpy()
    v[:] = np.ravel(a, order="F")
    return v, t


(rp, _1), (ci, _2), (va, _3), (hb, _4) = (pinned(csr.row_ptr), pinned(csr.col_idx),
                                          pinned(csr.values), pinned(cfg.rhs))
hb = hb.reshape(cfg.rhs.shape, order="F")
scfg = api.SolverConfig(variant="T", p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=2000)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A2 = api.CsrMatrix(ctx, csr.n, rp, ci, va)
    t1 = time.perf_counter()
    F2 = api.factorize(ctx, A2, scfg)
    t2 = time.perf_counter()
    xh, r, F2 = api.solve(A2, hb, it=it, F=F2)
    t3 = time.perf_counter()
    tf = F2.info["t_factorize"]
    del F2, A2
    t4 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} factorize wall {1e3*(t2-t1):.1f} (events {1e3*tf:.1f}) "
          f"solve wall {1e3*(t3-t2):.1f} (events {1e3*r.wall_time:.1f}) free {1e3*(t4-t3):.1f} "
          f"total {1e3*(t4-t0):.1f}", flush=True)

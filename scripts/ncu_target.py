"""Small fixed workload for ncu captures: one factorize + 3 preconditioner applies
(+ optional solve).  Usage: python scripts/ncu_target.py [config] [scale] [solve] [P]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
do_solve = len(sys.argv) > 3 and sys.argv[3] == "solve"
P = int(sys.argv[4]) if len(sys.argv) > 4 else None
ctx = api.Context(0)
cfg = configs.make_config(name, scale, P)
A = api.CsrMatrix.from_csr(ctx, cfg.system(0))  # c5: shift 0 (complex)
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
f = np.asfortranarray(cfg.rhs.astype(np.complex128) if cfg.shifts else cfg.rhs)
for _ in range(3):
    x = F.apply_precond_T(f)
if do_solve:
    api.solve(A, f, it=api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30), F=F)
ctx.synchronize()
print("ok", F.info["t_lu"], F.info["t_spikes"])

"""ncu target: config c5 (one shift, full size) factorize + 2 applies of the 16-RHS block."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
cfg = configs.make_config("c5", scale)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.system(0))
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
f = np.asfortranarray(cfg.rhs.astype(np.complex128))
for _ in range(2):
    x = F.apply_precond_T(f)
ctx.synchronize()
print("ok", F.info["t_lu"], f.shape)

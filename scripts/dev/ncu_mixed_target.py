"""ncu target: c3 P=64 with FP32 factor tiles, three one-column applies."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
cfg = configs.make_config("c3", scale, 64)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed,
                                           factor_fp32=True))
f = np.asfortranarray(cfg.rhs)
for _ in range(3):
    x = F.apply_precond_T(f)
ctx.synchronize()
print("ok")

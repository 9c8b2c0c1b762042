"""LU-only timing probe (development aid): Block-Jacobi factorize (band LU only) of a
config, repeated; prints the median t_lu and TF/s.  LRS_LIB selects a variant build.

  python scripts/lu_probe.py c2 [scale] [reps]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = configs.make_config(name, scale)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.system(0))
ts = []
for _ in range(reps):
    F = api.factorize(ctx, A, api.SolverConfig(variant="BJ", p=cfg.P, k=cfg.b, n_svd=0))
    ts.append(F.info["t_lu"])
    flops = F.info["lu_flops"]
    del F
ctx.set_profiling(True)
ctx.kernel_times(reset=True)
F = api.factorize(ctx, A, api.SolverConfig(variant="BJ", p=cfg.P, k=cfg.b, n_svd=0))
kt = ctx.kernel_times(reset=True)
t = float(np.median(ts))
print(json.dumps({"lib": os.environ.get("LRS_LIB", "default"), "config": name, "scale": scale,
                  "t_lu": t, "t_lu_all": ts, "tflops": flops / t / 1e12,
                  "profile_ms": {k: round(v[0], 2) for k, v in kt.items() if v[1]},
                  "update_tflops_profiled": None}), flush=True)

"""Per-kernel-class profile of one factorize (development aid).
  python scripts/setup_profile.py c4 0.25 [P]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
P = int(sys.argv[3]) if len(sys.argv) > 3 else None
cfg = configs.make_config(name, scale, P)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.system(0))
sc = api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
F = api.factorize(ctx, A, sc)
del F
ctx.set_profiling(True)
ctx.kernel_times(reset=True)
F = api.factorize(ctx, A, sc)
kt = ctx.kernel_times(reset=True)
print(json.dumps({"config": name, "scale": scale, "P": cfg.P, "r": cfg.r, "l": F.info["l"],
                  "t_lu": F.info["t_lu"], "t_spikes": F.info["t_spikes"],
                  "profile_ms": {k: [round(v[0], 2), v[1]] for k, v in kt.items() if v[1]}}))

"""The paper's mixed-precision configuration (single-precision preconditioner inside a double
Krylov solver; SPEC.md:539 `factor_fp32`) on a BASELINE config at full size:
factorize in FP64, keep an FP32 copy of the off-diagonal factor tiles for the applies, solve to
the config's tolerance (the true residual is formed in FP64).  Prints the FP64 run beside it.

  python scripts/run_mixed.py c3 1.0 64
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
from paper_2504_11167_b200 import api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
P = int(sys.argv[3]) if len(sys.argv) > 3 else None
cfg = configs.make_config(name, scale, P)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
S = cfg.matrix.to_scipy()
it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=4000)
with ClockSampler(0) as clk:
    for fp32 in (True, False, True):
        sc = api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed, factor_fp32=fp32)
        F = api.factorize(ctx, A, sc)
        x, rep, F = api.solve(A, cfg.rhs, it=it, F=F)
        res = float(np.linalg.norm(cfg.rhs[:, 0] - S @ x[:, 0]) / np.linalg.norm(cfg.rhs[:, 0]))
        print(json.dumps({"config": name, "scale": scale, "P": cfg.P, "factor_fp32": fp32,
                          "t_factorize": F.info["t_factorize"], "t_lu": F.info["t_lu"],
                          "t_spikes": F.info["t_spikes"], "t_solve": rep.wall_time,
                          "step_s": F.info["t_factorize"] + rep.wall_time,
                          "iterations": rep.iterations, "converged": rep.converged,
                          "residual_final": rep.residual_final, "host_residual": res,
                          "factor_bytes": F.info["factor_bytes"],
                          "apply_bytes": F.info["apply_bytes"],
                          "apply_ms": 1e3 * rep.wall_time / max(rep.precond_applications, 1)}),
              flush=True)
        del F
print(json.dumps({"clocks": clk.summary()}))

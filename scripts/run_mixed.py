"""The paper's timing configuration for the preconditioner (section 4.3: "the
preconditioners applied are single-precision variants"; SPEC.md:539 keeps it as a flag
with no acceptance weight): LR-SPIKE-T with FP32 off-diagonal factor tiles in the applies
(FP64 diagonal inverses, Krylov method, SpMV and interface algebra), on a BASELINE config,
against the committed FP64 oracle fixture of the same config.  Not the bench headline
(which measures the FP64 preconditioner); reported in DESIGN.md section 7.

  python scripts/run_mixed.py c3 1.0 64 tests/golden/c3_s1_P64.npz
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
from paper_2504_11167_b200 import api, configs  # noqa: E402

name, scale, P, fix = sys.argv[1], float(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
cfg = configs.make_config(name, scale, P)
xo = np.load(fix)["x"]
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
out = []
with ClockSampler(0) as clk:
    for fp32 in (False, True, True):
        F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed,
                                                   factor_fp32=fp32))
        it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=3000)
        x, rep, _ = api.solve(A, cfg.rhs, it=it, F=F)
        rel = float(np.linalg.norm(np.ravel(x) - np.ravel(xo)) / np.linalg.norm(xo))
        out.append({"factor_fp32": fp32, "t_factorize": F.info["t_factorize"],
                    "t_solve": rep.wall_time, "step": F.info["t_factorize"] + rep.wall_time,
                    "iterations": rep.iterations, "residual_final": rep.residual_final,
                    "rel_diff_vs_fp64_oracle": rel, "apply_bytes": F.info["apply_bytes"]})
        print(json.dumps(out[-1]), flush=True)
        del F
print(json.dumps({"clocks": clk.summary()}), flush=True)

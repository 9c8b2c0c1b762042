"""Run one BASELINE config end to end on the GPU and print a JSON summary.

  python scripts/run_config.py c3 [scale] [P] [shift]

The apply is timed on device-resident blocks of all RHS columns (CUDA events through
ctx.synchronize), with the per-kernel-class profile of one apply.  nvidia-smi clocks and
throttle reasons are sampled for the whole run (bench.ClockSampler) and reported as "clocks".
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
from paper_2504_11167_b200 import api, configs  # noqa: E402

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
P = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) > 0 else None
shift = int(sys.argv[4]) if len(sys.argv) > 4 else 0
t0 = time.perf_counter()
cfg = configs.make_config(name, scale, P)
tgen = time.perf_counter() - t0
ctx = api.Context(0)
t0 = time.perf_counter()
A = api.CsrMatrix.from_csr(ctx, cfg.system(shift))
tup = time.perf_counter() - t0
out = {"config": name, "scale": scale, "n": cfg.matrix.n, "nnz": cfg.matrix.nnz, "b": cfg.b,
       "P": cfg.P, "r": cfg.r, "method": cfg.method, "t_gen": tgen, "t_upload": tup}
clk = ClockSampler(0).__enter__()
try:
    t0 = time.perf_counter()
    F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
    out["t_factorize_wall"] = time.perf_counter() - t0
    inf = F.info
    out.update({k: inf[k] for k in ("t_factorize", "t_lu", "t_spikes", "lu_flops", "factor_bytes",
                                    "apply_bytes", "wl", "wu", "n_svd", "max_interface_cond")})
    out["lu_tflops"] = inf["lu_flops"] / inf["t_lu"] / 1e12
    import torch

    rhs = np.asfortranarray(cfg.rhs.astype(A.dtype))
    nc = rhs.shape[1]
    fd = torch.from_numpy(np.ascontiguousarray(rhs.T)).cuda().t()
    od = torch.empty_like(fd.t()).t()
    torch.cuda.synchronize()
    F.apply_precond_T(fd, od)
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        F.apply_precond_T(fd, od)
    ctx.synchronize()
    ta = (time.perf_counter() - t0) / 5
    out["apply_ncols"] = nc
    out["apply_ms"] = ta * 1e3
    out["apply_GBps_1col_model"] = inf["apply_bytes"] / ta / 1e9
    ctx.set_profiling(True)
    ctx.kernel_times(reset=True)
    F.apply_precond_T(fd, od)
    ctx.synchronize()
    out["apply_profile_ms"] = {k: round(v[0], 4) for k, v in ctx.kernel_times(reset=True).items()
                               if v[1]}
    ctx.set_profiling(False)
    it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=3000)
    t0 = time.perf_counter()
    x, rep, _ = api.solve(A, rhs, it=it, F=F)
    out["t_solve_wall"] = time.perf_counter() - t0
    out.update({"iterations": rep.iterations, "converged": rep.converged,
                "residual_final": rep.residual_final, "t_solve": rep.wall_time,
                "precond_applications": rep.precond_applications})
except api.Error as e:
    out["error"] = f"{type(e).__name__}: {e}"
finally:
    clk.__exit__(None, None, None)
out["clocks"] = clk.summary()
print(json.dumps(out), flush=True)

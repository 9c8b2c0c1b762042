"""Config c5 as specified (BASELINE.json configs[4]): all 8 FEAST contour shifts
z_j = 2 + 0.5 e^{i pi (2j+1)/8}, each system z_j I - A (complex128, n = 512,000, P = 16,
n_svd = 32) solved for the block of 16 RHS with GMRES(40) to 1e-10, one after the other on
one GPU (the shifts are independent systems: PAPER.md:1628; under torchrun bench.py
--config c5 runs them as replicas, one shift per rank).  Prints one JSON line per shift
(device times from the library's CUDA events) and a total, with the SM clocks sampled
during the run.

  python scripts/run_c5_shifts.py [scale] [shifts...]
  python scripts/run_c5_shifts.py [scale] conj

conj: A and the right-hand sides are real and the contour is symmetric about the real axis
(z_{7-j} = conj(z_j)), so (z_{7-j} I - A)^-1 b = conj((z_j I - A)^-1 b): shifts 0..3 are solved
and 4..7 are their conjugates -- the half-contour FEAST implementations use.  Every conjugated
solution is checked against its own system on the host (true relative residual per column).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
from paper_2504_11167_b200 import api, configs  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
conj = sys.argv[2:] == ["conj"]
shifts = list(range(4)) if conj else ([int(a) for a in sys.argv[2:]] or list(range(8)))
cfg = configs.make_config("c5", scale)
ctx = api.Context(0)
rhs = np.asfortranarray(cfg.rhs.astype(np.complex128))
tot = {"t_factorize": 0.0, "t_solve": 0.0}
with ClockSampler(0) as clk:
    for j in shifts:
        t0 = time.perf_counter()
        A = api.CsrMatrix.from_csr(ctx, cfg.system(j))
        F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
        it = api.IterConfig(tol=cfg.tol, method="gmres", restart=cfg.m, max_iters=4000)
        x, rep, _F = api.solve(A, rhs, it=it, F=F)
        wall = time.perf_counter() - t0
        out = {"shift": j, "z": [cfg.shifts[j].real, cfg.shifts[j].imag], "n": cfg.matrix.n,
               "P": cfg.P, "n_rhs": rhs.shape[1], "t_factorize": F.info["t_factorize"],
               "t_lu": F.info["t_lu"], "t_spikes": F.info["t_spikes"], "t_solve": rep.wall_time,
               "iterations": rep.iterations, "converged": rep.converged,
               "residual_final": rep.residual_final,
               "precond_applications": rep.precond_applications, "wall": wall}
        tot["t_factorize"] += out["t_factorize"]
        tot["t_solve"] += out["t_solve"]
        print(json.dumps(out), flush=True)
        if conj:  # shift 7 - j: the conjugate solution against its own system, on the host
            t1 = time.perf_counter()
            assert abs(cfg.shifts[7 - j] - np.conj(cfg.shifts[j])) < 1e-15
            Sj = cfg.system(7 - j).to_scipy()
            xc = np.conj(x)
            res = max(float(np.linalg.norm(rhs[:, c] - Sj @ xc[:, c]) / np.linalg.norm(rhs[:, c]))
                      for c in range(rhs.shape[1]))
            assert res <= cfg.tol * (1 + 1e-6), (7 - j, res)
            print(json.dumps({"shift": 7 - j, "from_conjugate_of": j, "residual_final": res,
                              "host_check_s": time.perf_counter() - t1}), flush=True)
        del F, _F, A, x  # the next shift's 106 GB of factors reuse this one's pool blocks
print(json.dumps({"total_8_shifts_s": tot["t_factorize"] + tot["t_solve"], **tot,
                  "conjugate_pairs": conj, "clocks": clk.summary()}), flush=True)

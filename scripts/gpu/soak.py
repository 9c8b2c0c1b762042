"""Race detection by repetition at full size (compute-sanitizer is closed on the pool): R
factorizations of a config, each followed by a one-column preconditioner apply and a 3-column
block solve on two partitions; every result must equal the first factorization's bit for bit
(the kernels are deterministic by construction, so an inter-CTA race -- mailbox words, TMEM
slot ring, TMA ring, cluster panels, the look-ahead streams, the copy stream of the Omega
upload -- shows as a bitwise difference).

  python scripts/gpu/soak.py c3 1.0 64 30"""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

name, scale, P, R = sys.argv[1], float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = configs.make_config(name, scale, P)
csr = cfg.system(0) if cfg.shifts else cfg.matrix
cplx = bool(cfg.shifts)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, csr)
sc = api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
rng = np.random.default_rng(7)


def rand(r, c):
    v = rng.uniform(-1, 1, (r, c))
    return np.asfortranarray(v + 1j * rng.uniform(-1, 1, (r, c)) if cplx else v)


f = rand(csr.n, 1)
ref = None
t0 = time.perf_counter()
diffs = 0
for it in range(R):
    F = api.factorize(ctx, A, sc)
    parts = [F.apply_precond_T(f)]
    for i in (0, cfg.P - 1):
        if it == 0 and i == 0:
            Rb = {}
        Rb.setdefault(i, rand(F.sizes[i], 3))
        parts.append(F.solve_block(i, Rb[i]))
        parts.append(F.solve_block_adjoint(i, Rb[i]))
    u, s, v = F.spike(0, api.SIDE_T)
    parts += [np.ascontiguousarray(s), np.ascontiguousarray(u)]
    h = [hashlib.sha256(np.ascontiguousarray(p).tobytes()).hexdigest() for p in parts]
    if ref is None:
        ref = h
    elif h != ref:
        diffs += 1
        print("DIFFERENCE at repetition", it, [a == b for a, b in zip(h, ref)], flush=True)
    del F
print(json.dumps({"config": name, "scale": scale, "P": cfg.P, "repetitions": R,
                  "bitwise_differences": diffs, "lu_sym": None, "wall_s": time.perf_counter() - t0,
                  "sha256_apply": ref[0][:16]}))
sys.exit(1 if diffs else 0)

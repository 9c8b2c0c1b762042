"""Setup-stage timing (development aid): factorize a config a few times, print the median
t_lu / t_spikes (LRS_LIB selects a variant build).  python scripts/setup_probe.py c2 [scale]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cfg = configs.make_config(name, scale)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.system(0))
lu, spk = [], []
for _ in range(4):
    F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
    lu.append(F.info["t_lu"])
    spk.append(F.info["t_spikes"])
    del F
print(json.dumps({"lib": os.environ.get("LRS_LIB", "default"), "config": name,
                  "t_lu": float(np.median(lu[1:])), "t_spikes": float(np.median(spk[1:])),
                  "t_spikes_all": spk}))

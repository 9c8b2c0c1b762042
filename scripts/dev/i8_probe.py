"""INT8-sliced vs DMMA trailing update (development aid): LU time and factor agreement.

  python scripts/i8_probe.py c2 [scale]
"""
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
out = {}
tiles = {}
for mode in ("0", "1", "0", "1"):
    os.environ["LRS_LU_I8"] = mode
    F = api.factorize(ctx, A, api.SolverConfig(variant="BJ", p=cfg.P, k=cfg.b, n_svd=0))
    out.setdefault(mode, []).append(F.info["t_lu"])
    flops = F.info["lu_flops"]
    tiles[mode] = [F.tiles(i) for i in range(min(cfg.P, 2))]
    del F
d = max(float(np.max(np.abs(a - b)) / max(np.max(np.abs(a)), 1e-300))
        for a, b in zip(tiles["0"], tiles["1"]))
print(json.dumps({"config": name, "scale": scale, "t_lu_dmma": out["0"], "t_lu_i8": out["1"],
                  "tflops_dmma": flops / min(out["0"]) / 1e12,
                  "tflops_i8": flops / min(out["1"]) / 1e12, "max_rel_tile_diff": d}), flush=True)

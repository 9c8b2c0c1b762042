"""The apply's one-RHS L and U sweeps run as ONE launch (band_solve_lu1_kernel: tickets of the
L sweep first, then the U sweep, whose tiles take their right-hand side from the L sweep's
mailbox words).  The arithmetic is the two-launch path's, so the preconditioner output and
a whole solve equal LRS_SOLVE_FUSED=0 bit for bit."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2504_11167_b200 import api, configs
name, scale, out = sys.argv[2], float(sys.argv[3]), sys.argv[4]
cfg = configs.make_config(name, scale)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
f = np.asfortranarray(configs.vector("uniform", 9, cfg.matrix.n))
y = F.apply_precond_T(f)
x, rep, _ = api.solve(A, cfg.rhs, it=api.IterConfig(tol=cfg.tol, method=cfg.method,
                                                   restart=cfg.m or 30, max_iters=500), F=F)
np.savez(out, y=y, x=x)
print(json.dumps({"hist": list(rep.residual_history), "it": rep.iterations}))
"""


@pytest.mark.parametrize("name,scale", [("c2", 24 / 64), ("c3", 24 / 96), ("c1", 96 / 256)])
def test_fused_lu_sweeps_bitwise(tmp_path, name, scale):
    res = {}
    for mode in ("1", "0"):
        out = str(tmp_path / f"r{mode}.npz")
        p = subprocess.run([sys.executable, "-c", CHILD, ROOT, name, str(scale), out],
                           env={**os.environ, "LRS_SOLVE_FUSED": mode}, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        res[mode] = (np.load(out), json.loads(p.stdout.strip().splitlines()[-1]))
    (a, ra), (b, rb) = res["1"], res["0"]
    assert np.array_equal(a["y"], b["y"]) and np.array_equal(a["x"], b["x"])
    assert ra == rb

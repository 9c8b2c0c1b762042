"""BiCGStab's t = A shat with its omega dots (t^H s, t^H t) runs as ONE fused kernel
(csrc/spmv.cu spmv_dot2_kernel): the chunk partials follow multidot_partial_kernel's row
order and reduction tree, so the fused solve must equal the unfused one (LRS_SPMV_DOT=0,
SpMV + multidot) bit for bit -- solution and residual history -- real and complex, one and
several right-hand sides."""
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
name, scale, nrhs, out = sys.argv[2], float(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
cfg = configs.make_config(name, scale)
ctx = api.Context(0)
A = api.CsrMatrix.from_csr(ctx, cfg.system(0))
dt = np.complex128 if cfg.shifts else np.float64
b = np.asfortranarray(configs.vector("uniform", 7, cfg.matrix.n, nrhs).astype(dt))
x, rep, F = api.solve(A, b, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed),
                      api.IterConfig(tol=1e-9, method="bicgstab", max_iters=400))
np.save(out, x)
print(json.dumps({"it": rep.iterations, "hist": list(rep.residual_history),
                  "launches": ctx.launches}))
"""


@pytest.mark.parametrize("name,scale,nrhs", [("c2", 24 / 64, 1), ("c2", 24 / 64, 3),
                                             ("c5", 0.3, 2)])
def test_fused_spmv_dot_bitwise(tmp_path, name, scale, nrhs):
    res = {}
    for mode in ("1", "0"):
        out = str(tmp_path / f"x{mode}.npy")
        p = subprocess.run([sys.executable, "-c", CHILD, ROOT, name, str(scale), str(nrhs), out],
                           env={**os.environ, "LRS_SPMV_DOT": mode}, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        res[mode] = (np.load(out), json.loads(p.stdout.strip().splitlines()[-1]))
    (x1, r1), (x0, r0) = res["1"], res["0"]
    assert np.array_equal(x1, x0)
    assert r1["hist"] == r0["hist"] and r1["it"] == r0["it"]
    assert r1["launches"] < r0["launches"]  # one dot kernel fewer per iteration

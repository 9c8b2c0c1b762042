"""Per-CTA timeline of the NR=1 band solves (development aid; needs a library built with
-DLRS_SOLVE_TRACE, selected by LRS_LIB, and LRS_STRACE=<output file>)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2504_11167_b200 import api, configs  # noqa: E402

cfg = configs.make_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = api.Context(0, st.cuda_stream)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
bd = torch.from_numpy(np.asfortranarray(cfg.rhs)).cuda()
xd = torch.empty_like(bd)
for _ in range(45):
    F.apply_precond_T(bd, xd)
torch.cuda.synchronize()
print("done")

"""Upload phases of the c3 CSR (LRS_UPLOAD_TRACE=1): pageable numpy arrays and page-locked
torch buffers, three uploads each."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2504_11167_b200 import api, configs  # noqa: E402

cfg = configs.make_config(sys.argv[1] if len(sys.argv) > 1 else "c3", 1.0, 64)
m = cfg.matrix
ctx = api.Context(0)


def pinned(a):
    t = torch.empty(a.size, dtype=torch.from_numpy(a[:0].copy()).dtype, pin_memory=True)
    v = t.numpy()
    v[:] = a
    return v, t


for tag, arrs in (("pageable", (m.row_ptr, m.col_idx, m.values)),
                  ("pinned", tuple(pinned(a) for a in (m.row_ptr, m.col_idx, m.values)))):
    rp, ci, va = (a[0] if isinstance(a, tuple) else a for a in arrs)
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A = api.CsrMatrix(ctx, m.n, rp, ci, va)
        print(tag, "upload %.1f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
        del A

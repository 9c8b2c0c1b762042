"""SpMV A/B on the c3 matrix (23.4M nnz): the shared-memory staged kernel (default) vs the
one-thread-per-row kernel (LRS_SPMV_SCALAR=1, run as a second process), CUDA events over
50 launches; algorithmic bytes nnz (8 + 4) + 4 (n + 1) + 2 n 8."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def measure():
    import numpy as np
    import torch

    from paper_2504_11167_b200 import api, configs

    cfg = configs.make_config("c3", 1.0, 64)
    ctx = api.Context(0)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    n, nnz = cfg.matrix.n, cfg.matrix.nnz
    x = torch.from_numpy(np.asfortranarray(cfg.rhs).T.copy()).cuda().t()
    y = torch.empty_like(x.t()).t()
    torch.cuda.synchronize()
    for _ in range(5):
        A.spmv(x, y)
    ctx.synchronize()
    ctx.set_profiling(True, classes=("spmv",))
    ctx.kernel_times(reset=True)
    for _ in range(50):
        A.spmv(x, y)
    ctx.synchronize()
    ms, cnt = ctx.kernel_times(reset=True)["spmv"]
    per = ms / cnt
    bytes_ = nnz * 12 + 4 * (n + 1) + 16 * n
    ref = cfg.matrix.to_scipy() @ cfg.rhs
    err = float(np.abs(y.cpu().numpy() - ref).max() / np.abs(ref).max())
    return {"kernel": "scalar" if os.environ.get("LRS_SPMV_SCALAR") == "1" else "staged",
            "ms": per, "GBps": bytes_ / per / 1e6, "bytes": bytes_, "max_rel_err": err}


if __name__ == "__main__":
    if len(sys.argv) > 1:
        print(json.dumps(measure()), flush=True)
    else:
        for env in ({}, {"LRS_SPMV_SCALAR": "1"}):
            out = subprocess.run([sys.executable, __file__, "one"], env={**os.environ, **env},
                                 capture_output=True, text=True)
            print(out.stdout.strip() or out.stderr[-2000:], flush=True)

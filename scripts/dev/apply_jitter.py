"""Distribution of single preconditioner-apply times (development aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2504_11167_b200 import api, configs  # noqa: E402

cfg = configs.make_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 300
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = api.Context(0, st.cuda_stream)
A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
bd = torch.from_numpy(np.asfortranarray(cfg.rhs)).cuda()
xd = torch.empty_like(bd)
for name, fn in (("T", F.apply_precond_T), ("BJ", F.apply_block_jacobi),
                 ("spmv", lambda a, b: A.spmv(a, b))):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(N)]
    for _ in range(5):
        fn(bd, xd)
    torch.cuda.synchronize()
    for e0, e1 in evs:
        e0.record(st)
        fn(bd, xd)
        e1.record(st)
    torch.cuda.synchronize()
    t = np.array([e0.elapsed_time(e1) for e0, e1 in evs])
    print(name, "ms p0 %.3f p10 %.3f p50 %.3f p90 %.3f p99 %.3f max %.3f mean %.3f" % (
        t.min(), *np.percentile(t, [10, 50, 90, 99]), t.max(), t.mean()), flush=True)
    big = np.flatnonzero(t > 1.3 * np.median(t))
    print("  slow idx", big[:40].tolist(), flush=True)
it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=2000)
for k in range(8):
    x, r, _ = api.solve(A, bd, it=it, F=F, x_out=xd)
    print("solve", r.iterations, r.precond_applications, "%.1f ms" % (1e3 * r.wall_time), flush=True)

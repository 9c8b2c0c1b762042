"""Quick perf probe of the GPU path on one config (development aid)."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
from paper_2504_11167_b200 import api, configs

name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
import torch
ctx = api.Context(0, torch.cuda.current_stream().cuda_stream)
print('dmma peak TF', ctx.dmma_peak_tflops(), flush=True)
t = time.time(); cfg = configs.make_config(name, scale); print('gen', time.time() - t, flush=True)
t = time.time(); A = api.CsrMatrix.from_csr(ctx, cfg.matrix); print('upload', time.time() - t, flush=True)
for rep in range(2):
    t = time.time()
    F = api.factorize(ctx, A, api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed))
    inf = F.info
    print('factorize wall', time.time() - t, {k: inf[k] for k in ('t_factorize', 't_lu', 't_spikes', 'lu_flops', 'factor_bytes', 'apply_bytes', 'wl', 'wu', 'max_interface_cond')}, flush=True)
    print('LU TF/s', inf['lu_flops'] / inf['t_lu'] / 1e12, flush=True)
import torch
f = torch.from_numpy(np.asfortranarray(cfg.rhs)).cuda()
x = torch.empty_like(f)
for bj in (False, True):
    fn = F.apply_block_jacobi if bj else F.apply_precond_T
    fn(f, x); torch.cuda.synchronize()
    t = time.time(); N = 10
    for _ in range(N): fn(f, x)
    torch.cuda.synchronize(); dt = (time.time() - t) / N
    print('apply', 'BJ' if bj else 'T', dt * 1e3, 'ms', inf['apply_bytes'] / dt / 1e9, 'GB/s', flush=True)
it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=1000)
t = time.time()
xs, r, _ = api.solve(A, cfg.rhs, it=it, F=F)
print('solve', time.time() - t, r.iterations, r.converged, r.residual_final, r.wall_time, r.precond_applications, flush=True)

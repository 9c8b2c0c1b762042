"""Command line driver (SPEC.md:544 `solve`, SPEC.md:131 `reorder`).

  python -m paper_2504_11167_b200.cli solve --in A.mtx [--rhs ones|uniform|B.mtx]
        [--variant t|i|otf|bj] [-p INT] [-k INT] [--nsvd INT] [--tol FLOAT] [--seed INT]
        [--method bicgstab|gmres|cg] [--restart INT] [--reorder] [--x-out x.npy]
        [--report out.json]
  python -m paper_2504_11167_b200.cli reorder --in A.mtx --out B.mtx [--report r.json]

`solve` reads the Matrix Market file, optionally applies the reorder pipeline (strip
disconnected rows, symmetric diagonal scaling, reverse Cuthill-McKee; the solution is mapped
back), factorizes and solves on the GPU, and writes the SPEC report
{variant, p, k, n_svd, iterations, inner_iterations, residual_final,
 comm:{stage:{messages, scalars}}, timings:{factorize, solve}, seed}.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np
import scipy.sparse as sp

from . import api, configs, reorder

_VARIANTS = {"t": "T", "i": "I", "otf": "OTF", "bj": "BJ"}


def _band(a) -> dict:
    S = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n)).tocoo()
    ku = int(np.max(S.col - S.row, initial=0))
    kl = int(np.max(S.row - S.col, initial=0))
    d = S.row == S.col
    tot = float(np.abs(S.data).sum())
    return {"n": int(a.n), "nnz": int(a.nnz), "ku": ku, "kl": kl, "k": max(ku, kl),
            "diag_weight": float(np.abs(S.data[d]).sum() / tot) if tot else 0.0,
            "band_density": float(a.nnz / ((ku + kl + 1) * a.n)) if a.n else 0.0}


def _pipeline(a):
    """strip -> scale -> RCM; returns (matrix, kept indices, scale, rcm forward)."""
    b, removed = reorder.strip_disconnected(a)
    keep = np.setdiff1d(np.arange(a.n), removed)
    b, d = reorder.diagonal_scale(b)
    f = reorder.rcm_ordering(b)
    return reorder.apply_permutation(b, f, f), keep, d, f


def cmd_reorder(args) -> int:
    a = reorder.read_matrix_market(args.inp)
    b, keep, d, f = _pipeline(a)
    reorder.write_matrix_market(args.out, b)
    rep = {"before": _band(a), "after": _band(b), "removed": int(a.n - keep.size)}
    if args.report:
        with open(args.report, "w") as fh:
            json.dump(rep, fh, indent=2)
    print(json.dumps(rep))
    return 0


def cmd_solve(args) -> int:
    a = reorder.read_matrix_market(args.inp)
    n = a.n
    if args.rhs == "ones":
        f = np.ones((n, 1))
    elif args.rhs == "uniform":
        f = configs.vector("uniform", args.seed, n)
    else:
        B = reorder.read_matrix_market(args.rhs)
        f = sp.csr_matrix((B.values, B.col_idx, B.row_ptr), shape=(B.n, int(B.col_idx.max(initial=0)) + 1)).toarray()
        if f.shape[0] != n:
            raise api.DimensionError("rhs rows must equal n")
    f = np.asfortranarray(f, dtype=np.float64)
    m = a
    keep = d = fwd = None
    if args.reorder:
        m, keep, d, fwd = _pipeline(a)
        # scaled, permuted system: (D A D) y = D f,  x = D y on the kept rows
        g = f[keep] * d[:, None]
        gp = np.empty_like(g)
        gp[fwd] = g
        rhs = np.asfortranarray(gp)
    else:
        rhs = f
    ctx = api.Context(args.device)
    A = api.CsrMatrix(ctx, m.n, m.row_ptr, m.col_idx, m.values)
    k = args.k if args.k else A.band_metrics().k
    cfg = api.SolverConfig(variant=_VARIANTS[args.variant], p=args.p, k=k, n_svd=args.nsvd,
                           seed=args.seed, spike_mode=args.spike_mode)
    it = api.IterConfig(tol=args.tol, method=args.method, restart=args.restart,
                        max_iters=args.max_iters)
    t0 = time.perf_counter()
    F = api.factorize(ctx, A, cfg)
    t_fact = time.perf_counter() - t0
    x, rep, _ = api.solve(A, rhs, it=it, F=F)
    xs = np.asarray(x)
    if args.reorder:
        y = xs[fwd] * d[:, None]
        xs = np.zeros_like(f)
        xs[keep] = y
        # the stripped rows are decoupled: a_ii x_i = f_i
        S = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(n, n))
        dropped = np.setdiff1d(np.arange(n), keep)
        xs[dropped] = f[dropped] / S.diagonal()[dropped][:, None]
    S = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(n, n))
    res = float(np.max(np.linalg.norm(S @ xs - f, axis=0) / np.maximum(np.linalg.norm(f, axis=0), 1e-300)))
    report = {"variant": args.variant, "p": args.p, "k": int(k), "n_svd": int(F.n_svd),
              "iterations": rep.iterations, "inner_iterations": rep.inner_iterations,
              "residual_final": res, "converged": rep.converged,
              "comm": {s: {"messages": int(v[0]), "scalars": int(v[1])} for s, v in rep.comm.items()},
              "timings": {"factorize": t_fact, "solve": rep.wall_time}, "seed": args.seed,
              "reordered": bool(args.reorder), "band": _band(m)}
    if args.x_out:
        np.save(args.x_out, xs)
    if args.report:
        with open(args.report, "w") as fh:
            json.dump(report, fh, indent=2)
    print(json.dumps(report))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="lrspike")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve")
    s.add_argument("--in", dest="inp", required=True)
    s.add_argument("--rhs", default="ones")
    s.add_argument("--variant", default="t", choices=sorted(_VARIANTS))
    s.add_argument("-p", type=int, default=4)
    s.add_argument("-k", type=int, default=0)
    s.add_argument("--nsvd", type=int, default=8)
    s.add_argument("--tol", type=float, default=1e-8)
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--spike-mode", default="spike", choices=["spike", "coupling"],
                   help="spike construction: randomized SVD of the spike (SPEC.md:286) or "
                        "truncated SVD of the coupling blocks (north_star setup (1))")
    s.add_argument("--method", default="bicgstab", choices=["bicgstab", "gmres", "cg"])
    s.add_argument("--restart", type=int, default=30)
    s.add_argument("--max-iters", type=int, default=1000)
    s.add_argument("--reorder", action="store_true")
    s.add_argument("--device", type=int, default=0)
    s.add_argument("--x-out", default=None)
    s.add_argument("--report", default=None)
    r = sub.add_parser("reorder")
    r.add_argument("--in", dest="inp", required=True)
    r.add_argument("--out", required=True)
    r.add_argument("--report", default=None)
    args = ap.parse_args(argv)
    return cmd_solve(args) if args.cmd == "solve" else cmd_reorder(args)


if __name__ == "__main__":
    sys.exit(main())

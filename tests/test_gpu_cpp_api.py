"""The C++ drop-in API (include/lrspike) on the GPU against oracle fixtures.

The oracle (CPU checker) computes, on the c1 structure (48 x 48 grid, P = 4, k = 48,
n_svd = 8) and the c5 structure (complex128, 16^3 grid, P = 4, 2 RHS):
randomized_spike_svd (both sides) and the coupling-mode spike, the truncated
preconditioner and matvec_lowrank from its own spikes, the exact reduced matvec, and the
BiCGStab / GMRES solutions; tests/cpp/test_api (C++ -> C-ABI -> GPU) recomputes each of
them through the C++ API -- randomized_spike_svd / spike_tips, build_truncated_precond /
apply_truncated_precond / matvec_lowrank from explicit spikes, matvec_exact, bicgstab /
gmres on operator contracts, spmv without re-upload, factorize_dist on a one-rank
in-library NCCL communicator, and a complex128 GMRES solve -- and checks the bars it prints.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import configs

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_api")


class _Writer:
    def __init__(self, d):
        self.d = d
        self.lines = []

    def put(self, name, a, extra=0):
        a = np.asarray(a)
        if a.ndim == 1:
            a = a.reshape(-1, 1)
        kind = {np.dtype(np.float64): "f64", np.dtype(np.complex128): "c128",
                np.dtype(np.int64): "i64"}[a.dtype]
        np.asfortranarray(a).ravel(order="F").tofile(os.path.join(self.d, name + ".bin"))
        self.lines.append(f"{name} {a.shape[0]} {a.shape[1]} {kind} {int(extra)}")

    def close(self):
        with open(os.path.join(self.d, "manifest.txt"), "w") as fh:
            fh.write("\n".join(self.lines) + "\n")


def _pack(xt, xb):
    return np.concatenate([np.concatenate([t, b]) for t, b in zip(xt, xb)])


def _unpack(v, p, k):
    return [v[2 * k * i:2 * k * i + k] for i in range(p)], [v[2 * k * i + k:2 * k * (i + 1)]
                                                             for i in range(p)]


def _usv(s):
    return (s.u * s.sigma) @ s.v


def make_fixtures(d):
    w = _Writer(d)
    c = configs.make_config("c1", 48 / 256)
    S = c.matrix.to_scipy()
    p, k, r, seed = c.P, c.b, c.r, c.seed
    os_ = (r + 1) // 2
    w.put("A_rowptr", c.matrix.row_ptr, p)
    w.put("A_colidx", c.matrix.col_idx, k)
    w.put("A_values", c.matrix.values, r)
    w.put("rhs", c.rhs, seed)
    lay = O.make_layout(S.shape[0], p, k)
    bl = O.extract_blocks(S, lay)
    f0, f1 = O.factorize_block(bl.A[0]), O.factorize_block(bl.A[1])
    sT = O.randomized_spike_svd(f0, bl.B[0], O.SIDE_T, r, os_, 2, seed, 0)
    w.put("usvT0", _usv(sT))
    w.put("sigT0", sT.sigma)
    w.put("usvW1", _usv(O.randomized_spike_svd(f1, bl.C[1], O.SIDE_W, r, os_, 2, seed, 1)))
    w.put("usvC0", _usv(O.coupling_spike_svd(f0, bl.B[0], O.SIDE_T, r, os_, 2, seed, 0)))
    cfg = O.SolverConfig(variant="T", p=p, k=k, n_svd=r, seed=seed)
    F = O.factorize(S, cfg)
    for i in range(p - 1):
        w.put(f"uT{i}", F.spT[i].u)
        w.put(f"vT{i}", F.spT[i].v)
        w.put(f"sT{i}", F.spT[i].sigma)
        w.put(f"uW{i + 1}", F.spW[i + 1].u)
        w.put(f"vW{i + 1}", F.spW[i + 1].v)
        w.put(f"sW{i + 1}", F.spW[i + 1].sigma)
    g = np.random.default_rng(11).uniform(-1, 1, (2 * k * p, 2))
    w.put("g", g)
    top, bot = _unpack(g, p, k)
    w.put("trunc_g", _pack(*O.apply_truncated_precond(F.trunc, top, bot)))
    w.put("lowrank_g", _pack(*O.matvec_lowrank(F, top, bot)))
    w.put("exact_g", _pack(*O.matvec_otf(F, top, bot)))
    for method in ("bicgstab", "gmres"):
        x, rep, _ = O.solve(S, c.rhs, cfg, O.IterConfig(tol=1e-8, restart=30), method=method, F=F)
        w.put(f"x_{method}", x, rep.iterations)
    # complex128: c5 structure, shift 2, 2 RHS
    z = configs.make_config("c5", 16 / 80, P=4)
    Zm = z.system(2)
    Zs = Zm.to_scipy()
    rhs = np.asfortranarray(z.rhs[:, :2].astype(np.complex128))
    w.put("Z_rowptr", Zm.row_ptr, z.P)
    w.put("Z_colidx", Zm.col_idx, z.b)
    w.put("Z_values", Zm.values, z.r)
    w.put("zrhs", rhs, z.seed)
    zcfg = O.SolverConfig(variant="T", p=z.P, k=z.b, n_svd=z.r, seed=z.seed)
    zx, zrep, ZF = O.solve(Zs, rhs, zcfg, O.IterConfig(tol=1e-10, restart=40), method="gmres")
    w.put("zx", zx, zrep.iterations)
    w.put("zusvT0", _usv(ZF.spT[0]))
    w.close()


def test_cpp_api_ops_against_oracle(tmp_path):
    make_fixtures(str(tmp_path))
    r = subprocess.run([EXE, "oracle", str(tmp_path)], capture_output=True, text=True,
                       timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
